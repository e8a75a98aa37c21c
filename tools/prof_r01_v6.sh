set -x
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p6_plain.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p6_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p6_ncu_list.log 2>&1; echo list rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_conceal -s 3 -c 1 -o gpurun_out/prof_r01_v6_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p6_ncu_full.log 2>&1; echo full rc=$?
