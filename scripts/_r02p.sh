set -x
python scripts/prof_cfg.py C3 65536 8 > gpurun_out/r02p_c3_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 20 -c 1 \
  -o gpurun_out/r02p_move_c3 -f python scripts/prof_cfg.py C3 65536 8 > gpurun_out/r02p_ncu_c3.log 2>&1
python scripts/prof_cfg.py C5 65536 20 > gpurun_out/r02p_c5_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 20 -c 1 \
  -o gpurun_out/r02p_move_c5 -f python scripts/prof_cfg.py C5 65536 20 > gpurun_out/r02p_ncu_c5.log 2>&1
for s in "" "8,20"; do SPECMC_SHAPE=$s python scripts/probe.py C3:131072 >> gpurun_out/r02p_shape_c3.log 2>&1; done
echo done
