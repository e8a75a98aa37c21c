# Round-1 evidence run: bench lines (ours, reference arm, cfg4 forced HQL/IDL),
# the ncu launch list of the default bench command, and one ncu --set full
# capture of k_conceal on the default workload.  Each ncu pass runs only after
# the same command exited 0 without ncu.
set -x
python bench.py > gpurun_out/f_bench.log 2>&1; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.log 2>&1; echo ref rc=$?
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg4.log 2>&1; echo cfg4 rc=$?
python bench.py --workload cfg4idl --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg4idl.log 2>&1; echo cfg4idl rc=$?
python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg2.log 2>&1; echo cfg2 rc=$?
python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg1.log 2>&1; echo cfg1 rc=$?
python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg3.log 2>&1; echo cfg3 rc=$?
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_plain.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_list.log 2>&1; echo list rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_conceal -s 3 -c 1 -o gpurun_out/prof_r01_final_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_full.log 2>&1; echo full rc=$?
