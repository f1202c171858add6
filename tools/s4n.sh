mkdir -p gpurun_out/s4n
timeout 900 python -m pytest tests/test_gpu_mdp.py -q -x > gpurun_out/s4n/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4n/t.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
MDP_N=10000 python tools/mdp_variants.py paper_2511_13724_b200/libseneca.so variants/mdp_d1.so
