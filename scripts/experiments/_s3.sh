# session-2 pass 1: gpu tests on the new lib, A/B base vs uniform-grid Shirley, one ncu capture of the new move kernel
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/s3_gputests.log
timeout 900 python scripts/ab.py 3 C2:full,C1:full,C4x64:full paper_2604_03271_b200/lib_base.so paper_2604_03271_b200/lib_uni.so > gpurun_out/s3_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s3_ab.log | grep -v clocks
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 30 -c 1 -o gpurun_out/s3_move -f python scripts/prof_c2.py 65536 10 > gpurun_out/s3_ncu.log 2>&1; echo "ncu rc=$?"
