timeout 2400 python scripts/ab.py 2 C2:full,C1:full,C4x64:full,C3:65536 paper_2604_03271_b200/lib_b0.so paper_2604_03271_b200/lib_b1.so paper_2604_03271_b200/lib_b2.so > gpurun_out/s16_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s16_ab.log | grep -v clocks
