timeout 900 python -m pytest tests/test_gpu_ods.py -q -x -k "signal_paths" 2>&1 | tail -3
