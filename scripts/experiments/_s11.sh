timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s11_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/s11_gputests.log
for L in lib_v9.so lib_v10.so; do SPECMC_LIB=paper_2604_03271_b200/$L timeout 300 python scripts/e2e_probe2.py > gpurun_out/s11_e2e_$L.log 2>&1; echo $L; cat gpurun_out/s11_e2e_$L.log; done
timeout 600 python bench.py > gpurun_out/s11_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s11_bench.log
