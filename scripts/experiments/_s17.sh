# grid-level tempering for T = 65536 (C2): threshold / slice-length sweep
for cfg in "" "SPECMC_GRID_T=32768 SPECMC_SLICE=16384" "SPECMC_GRID_T=32768 SPECMC_SLICE=8192" "SPECMC_GRID_T=32768 SPECMC_SLICE=4096" "SPECMC_GRID_T=32768 SPECMC_SLICE=2048"; do
  for r in 1 2; do echo "[$cfg]"; env $cfg python scripts/probe.py C2:full | grep -v clocks; done
done
