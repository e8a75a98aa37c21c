# phase cycles per kernel build on the narrow-DAG configs (diag build)
export BM_NATIVE_VARIANT=diag
for kb in 512 cluster; do
  python tools/phases.py 1 1 sentinel $kb > gpurun_out/g_ph_cfg1_$kb.log 2>&1; echo cfg1 $kb rc=$?
  python tools/phases.py 3 16 efficient $kb > gpurun_out/g_ph_cfg3_$kb.log 2>&1; echo cfg3 $kb rc=$?
done
