set -x
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize.py > gpurun_out/san_racecheck.log 2>&1; echo racecheck rc=$?
tail -5 gpurun_out/san_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_synccheck.log 2>&1; echo synccheck rc=$?
tail -5 gpurun_out/san_synccheck.log
