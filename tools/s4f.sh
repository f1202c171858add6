mkdir -p gpurun_out/s4f
bash tools/phase_ab.sh s4f imagenet1k 5000 1 base fast3t > gpurun_out/s4f/phases.txt
cat gpurun_out/s4f/phases.txt
