# Round-2 measurement pass on one B200 (run under gpurun; outputs in gpurun_out/):
# GPU tests, bench lines for C1-C5, C2 launch list and one --set full capture
# of the C2 move kernel.  usage: bash scripts/r02_measure.sh TAG [quick]
TAG=$1
free -g > gpurun_out/${TAG}_host_mem.txt; nproc >> gpurun_out/${TAG}_host_mem.txt
python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/${TAG}_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c2.log 2>&1
python bench.py --config C1 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c1.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/prof_c2.py 65536 10 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 30 -c 1 \
  -o gpurun_out/${TAG}_move -f python scripts/prof_c2.py 65536 10 > /dev/null 2>&1
if [ "$2" != "quick" ]; then
  python bench.py --config C4 --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_c4.log 2>&1
  python bench.py --config C5 --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_c5.log 2>&1
  python bench.py --config C3 --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_c3.log 2>&1
fi
echo done
