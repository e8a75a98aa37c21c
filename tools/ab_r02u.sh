# round 2: the next patch's pick in the warp-0 segment that commits the patch before it (BM_PICK_MERGE)
# (bit-identical) (dev A/B); prev = the commit before
python tools/bitcmp.py base prev 5 8 256 > gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 1 1 >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 3 2 cluster >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 4 1 >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 5 8 512 >> gpurun_out/u_bit.log 2>&1
python tools/bitcmp.py base prev 2 1 >> gpurun_out/u_bit.log 2>&1
grep cfg gpurun_out/u_bit.log
timeout 600 python -m pytest tests/test_gpu.py -q -m gpu -p no:cacheprovider -k "total_loss or golden or flat_block or periodic" 2>&1 | tail -1
bash tools/ab.sh cfg5 3 base prev base prev
bash tools/ab.sh cfg4idl 3 base prev
bash tools/ab.sh cfg2 10 base prev
bash tools/ab.sh cfg3 3 base prev
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/u_phases_cfg5.txt 2>&1; grep "per-patch\|idl_" gpurun_out/u_phases_cfg5.txt
