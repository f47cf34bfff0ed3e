timeout 1500 python scripts/ab.py 2 C4x64:full,C4x256:4096,C2:full paper_2604_03271_b200/lib_e0.so paper_2604_03271_b200/lib_e1.so > gpurun_out/s23_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s23_ab.log | grep -v clocks
