# round 2: cluster build's k-nearest merge by rank (one DSMEM round trip), FP64 cell publish only with readers (dev A/B)
python tools/bitcmp.py base prev 1 1 > gpurun_out/n_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/n_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 256 >> gpurun_out/n_bit.log 2>&1
python tools/bitcmp.py base prev 5 32 cluster >> gpurun_out/n_bit.log 2>&1
grep cfg gpurun_out/n_bit.log
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fullframe.py -q -m gpu -p no:cacheprovider > gpurun_out/n_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/n_tests.log
bash tools/ab.sh cfg1 10 base prev base prev
bash tools/ab.sh cfg3 3 base prev
bash tools/ab.sh cfg2 10 base prev
bash tools/ab.sh cfg5 3 base prev
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_conceal -c 1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/n_dram.log 2>&1; grep -E "dram__bytes" gpurun_out/n_dram.log
