timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s9_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/s9_gputests.log
timeout 2000 python scripts/ab.py 2 C2:full,C1:full,C4x64:full,C3:65536,C5:16384 paper_2604_03271_b200/lib_v4.so paper_2604_03271_b200/lib_v7_384.so paper_2604_03271_b200/lib_v7_512.so > gpurun_out/s9_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s9_ab.log | grep -v clocks
for L in lib_v4.so lib_v7_512.so; do SPECMC_LIB=paper_2604_03271_b200/$L timeout 300 python scripts/e2e_probe2.py > gpurun_out/s9_e2e_$L.log 2>&1; echo $L; cat gpurun_out/s9_e2e_$L.log; done
