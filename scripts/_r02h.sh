python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h_gputests.log 2>&1
echo "rc=$?" >> gpurun_out/r02h_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02h_smoke.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_c2.log 2>&1
echo done
