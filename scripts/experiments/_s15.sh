timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s15_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/s15_gputests.log
SPECMC_TRACE=1 timeout 300 python scripts/e2e_probe3.py 2>&1 | grep -v "~ClassRun\|~Arena" | tail -14
timeout 600 python bench.py > gpurun_out/s15_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s15_bench.log
