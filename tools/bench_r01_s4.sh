# Round-1 (session 2, final) bench lines: the default bench (cfg5, CPU baseline, e2e),
# the reference arm, and the other configs (cfg4 forced HQL / IDL, cfg1-3).
set -x
python bench.py > gpurun_out/b4_bench.log 2>&1; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b4_ref.log 2>&1; echo ref rc=$?
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_cfg4.log 2>&1; echo cfg4 rc=$?
python bench.py --workload cfg4idl --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_cfg4idl.log 2>&1; echo cfg4idl rc=$?
python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_cfg3.log 2>&1; echo cfg3 rc=$?
python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4_cfg2.log 2>&1; echo cfg2 rc=$?
python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4_cfg1.log 2>&1; echo cfg1 rc=$?
