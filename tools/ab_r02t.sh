# round 2: beta epilogue residual divisions (BM_BETA_PAR) and covariance epilogue divisions (BM_COV_PAR) on all
# threads (bit-identical) (dev A/B); prev = the commit before, nobp / nocp = base without one of them
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/t_bit.log 2>&1
grep cfg gpurun_out/t_bit.log
bash tools/ab.sh cfg5 3 base prev nobp nocp base prev
bash tools/ab.sh cfg4 3 base prev nobp nocp
bash tools/ab.sh cfg1 10 base prev
bash tools/ab.sh cfg3 3 base prev
