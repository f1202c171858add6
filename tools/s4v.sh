timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 python __graft_entry__.py smoke 2>&1 | grep -E "smoke ok|ERROR" | head -5; echo "ncu smoke rc=${PIPESTATUS[0]}"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ods_rounds -c 2 python tools/profile_ods.py imagenet1k 200 --plain 2>&1 | grep -E "ERROR|gpu__time" | head -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_ods.py -q -x -k "toy or cold" 2>&1 | tail -1
