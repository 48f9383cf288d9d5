# compute-sanitizer on two small K7 launches (memcheck, then racecheck on shared memory).
mkdir -p gpurun_out/r2br
timeout 300 python tools/k7_small.py 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck python tools/k7_small.py > gpurun_out/r2br/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -6 gpurun_out/r2br/memcheck.log
timeout 900 compute-sanitizer --tool racecheck python tools/k7_small.py > gpurun_out/r2br/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -8 gpurun_out/r2br/racecheck.log
