# usage: bash scripts/_ncu_full.sh CFG LIB...  -- plain run, then one --set full capture of a move launch per lib
CFG=$1; shift
for L in "$@"; do
  SPECMC_LIB=paper_2604_03271_b200/$L python scripts/probe.py $CFG > gpurun_out/plain_$L.log 2>&1 && \
  SPECMC_LIB=paper_2604_03271_b200/$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 20 -c 1 -o gpurun_out/full_$L -f python scripts/probe.py $CFG > gpurun_out/ncu_full_$L.log 2>&1
  echo "$L rc=$?"
done
