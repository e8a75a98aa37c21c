# round 2: LOO row tiles per pass with y0 from shared memory and the split weight/sum structure (dev A/B)
python tools/bitcmp.py base srr2 5 8 256 > gpurun_out/m_bit.log 2>&1
python tools/bitcmp.py base srr3 4 1 256 >> gpurun_out/m_bit.log 2>&1
grep cfg gpurun_out/m_bit.log
bash tools/ab.sh cfg5 3 base y0s srr2 srr3 base
bash tools/ab.sh cfg4 3 base srr2 srr3
