CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_mdp2.py variants/mdp_d2.so
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_mdp2.py paper_2511_13724_b200/libseneca.so
