set -x
bash tools/ab.sh cfg5 5 r0 base r0 base
python tests/../tools/gpu_check.py > gpurun_out/ab1_golden.txt 2>&1; tail -3 gpurun_out/ab1_golden.txt
