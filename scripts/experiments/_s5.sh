# A/B uni vs v3 (P in smem for W=2, 512-thread CTAs, split noise partials, B recurrence, endpoint in place)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s5_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/s5_gputests.log
timeout 1200 python scripts/ab.py 3 C2:full,C1:full,C4x64:full,C3:65536,C5:16384 paper_2604_03271_b200/lib_uni.so paper_2604_03271_b200/lib_v3.so > gpurun_out/s5_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s5_ab.log | grep -v clocks
SPECMC_LIB=paper_2604_03271_b200/lib_v3.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 30 -c 1 -o gpurun_out/s5_move -f python scripts/prof_c2.py 65536 10 > gpurun_out/s5_ncu.log 2>&1; echo "ncu rc=$?"
