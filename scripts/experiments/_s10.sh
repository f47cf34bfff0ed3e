timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s10_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/s10_gputests.log
timeout 2400 python scripts/ab.py 2 C2:full,C1:full,C4x64:full,C3:65536,C5:16384 paper_2604_03271_b200/lib_v4.so paper_2604_03271_b200/lib_v8.so paper_2604_03271_b200/lib_v9.so > gpurun_out/s10_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s10_ab.log | grep -v clocks
