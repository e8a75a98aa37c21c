python tools/cli_case_debug.py > gpurun_out/c2_cli.log 2>&1; echo cli rc=$?
timeout 900 python -m pytest tests/test_cli_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/c2_clitest.log 2>&1; echo clitest rc=$?
python tools/scale_sim.py 32 256 > gpurun_out/c2_scale.log 2>&1; echo scale rc=$?
python tools/critical_path.py cfg3 > gpurun_out/c2_cp_cfg3.log 2>&1; echo cp rc=$?
BM_NATIVE_VARIANT=diag python tools/phases.py 5 256 efficient > gpurun_out/c2_phases_cfg5.log 2>&1; echo ph rc=$?
BM_NATIVE_VARIANT=diag python tools/phases.py 3 16 efficient > gpurun_out/c2_phases_cfg3.log 2>&1; echo ph3 rc=$?
