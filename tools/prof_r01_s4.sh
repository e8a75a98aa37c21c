# Round-1 (session 2) evidence: ncu launch list of the default bench command and
# one ncu --set full capture of k_conceal on the default workload (cfg5).  Each
# ncu pass runs only after the same command exited 0 without ncu.
set -x
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p4_plain.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p4_ncu_list.log 2>&1; echo list rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:_ZN2bm9k_conceal -s 3 -c 1 -o gpurun_out/prof_r01_s4_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p4_ncu_full.log 2>&1; echo full rc=$?
