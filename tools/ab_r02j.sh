# round 2: gate first-chunk prefetch, LOO two row tiles per pass (dev A/B)
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/j_bit.log 2>&1
python tools/bitcmp.py base rr2 5 8 256 >> gpurun_out/j_bit.log 2>&1
grep cfg gpurun_out/j_bit.log
bash tools/ab.sh cfg5 3 base prev nopre rr2 base prev
bash tools/ab.sh cfg4 3 base rr2 prev
bash tools/ab.sh cfg4idl 5 base nopre
