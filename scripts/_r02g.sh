python bench.py --config C1 --steps 5 --warmup 3 > gpurun_out/r02g_bench_c1.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_bench_c2.log 2>&1
python -m pytest tests/test_cpp_adapter.py -q -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_tests.log
echo done
