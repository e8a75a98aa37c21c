# round 2: rolled L^-1 substitution (BM_LINV_ROLL), alpha den/num pairwise sums on 8-lane groups (BM_ALPHA_PAR)
# (bit-identical) (dev A/B); prev = 958d365, nolr = base without BM_LINV_ROLL
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/t_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/t_bit.log 2>&1
grep cfg gpurun_out/t_bit.log
bash tools/ab.sh cfg5 3 base prev nolr base prev
bash tools/ab.sh cfg4 3 base prev nolr
bash tools/ab.sh cfg1 10 base prev
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/t_phases_cfg5.txt 2>&1; head -16 gpurun_out/t_phases_cfg5.txt
