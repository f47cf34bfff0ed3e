python scripts/ab.py 3 C2:65536,C3:131072,C5:65536 scripts/lib_base.so paper_2604_03271_b200/libspecmc_b200.so > gpurun_out/r02q_ab.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_coherence.py -q -x -p no:cacheprovider > gpurun_out/r02q_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02q_tests.log
echo done
