timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s8_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/s8_gputests.log
timeout 1500 python scripts/ab.py 3 C2:full,C1:full,C4x64:full paper_2604_03271_b200/lib_v4.so paper_2604_03271_b200/lib_v6a.so paper_2604_03271_b200/lib_v6b.so > gpurun_out/s8_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s8_ab.log | grep -v clocks
