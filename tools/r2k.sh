#!/bin/bash
T=${1:-r2k}; mkdir -p gpurun_out/$T
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mdp_sweep -s 1 -c 1 -o gpurun_out/$T/mdp10k \
  python tools/profile_mdp.py 10000 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_lines.py gpurun_out/$T/mdp10k.ncu-rep 70 --by-inst > gpurun_out/$T/lines_inst.txt 2>&1
python tools/ncu_lines.py gpurun_out/$T/mdp10k.ncu-rep 50 > gpurun_out/$T/lines_stall.txt 2>&1
ncu -i gpurun_out/$T/mdp10k.ncu-rep --page raw --csv > gpurun_out/$T/raw.csv 2>&1
rm -f gpurun_out/$T/*.ncu-rep
