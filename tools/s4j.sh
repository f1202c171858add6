for n in 10000 100000; do MDP_N=$n python tools/mdp_variants.py variants/mdp_base.so variants/mdp_blk.so variants/mdp_base.so variants/mdp_blk.so; done
