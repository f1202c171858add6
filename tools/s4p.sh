for n in 10000 100000; do MDP_N=$n python tools/mdp_variants.py variants/mdp_d2.so variants/mdp_cap2.so variants/mdp_minb2.so variants/mdp_d2.so variants/mdp_cap2.so variants/mdp_minb2.so; done
