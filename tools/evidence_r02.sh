# Round-2 evidence run ($1 = tag): GPU suite, bench lines (ours, reference arm,
# cfg1-4/cfg4idl), the ncu launch list of the default bench command and one
# ncu --set full capture of k_conceal.  Each ncu pass runs only after the same
# command exited 0 without ncu.
T=${1:-r02}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/${T}_tests.log
python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/${T}_bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.log 2>&1; echo ref rc=$?
for w in cfg1 cfg2 cfg3 cfg4 cfg4idl; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_$w.log 2>&1; echo $w rc=$?
done
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_plain.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_list.log 2>&1; echo list rc=$?
if [ -n "$FULL" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_conceal -s 3 -c 1 -o gpurun_out/prof_${T}_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_full.log 2>&1; echo full rc=$?
fi
