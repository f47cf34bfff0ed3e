# Full measurement pass for one round: bench line, launch list, one --set full capture of the move kernel.
# usage: bash scripts/_prof_round.sh TAG
TAG=$1
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/${TAG}_plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e > gpurun_out/${TAG}_ncu1.log 2>&1
python scripts/prof_c2.py 65536 10 > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_chain -s 30 -c 1 -o gpurun_out/${TAG}_move -f python scripts/prof_c2.py 65536 10 > gpurun_out/${TAG}_ncu2.log 2>&1
echo "done $?"; tail -1 gpurun_out/${TAG}_bench.log
