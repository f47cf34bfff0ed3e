# session-2 pass 2: gpu tests on v2 (fold Lorentzian amplitude into rcp, paired noise layout), A/B uni vs v2, ncu of v2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/s4_gputests.log
timeout 900 python scripts/ab.py 3 C2:full,C1:full,C4x64:full paper_2604_03271_b200/lib_uni.so paper_2604_03271_b200/lib_v2.so > gpurun_out/s4_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s4_ab.log | grep -v clocks
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 30 -c 1 -o gpurun_out/s4_move -f python scripts/prof_c2.py 65536 10 > gpurun_out/s4_ncu.log 2>&1; echo "ncu rc=$?"
