mkdir -p gpurun_out/prof
MO_B200_JTJ=tma MO_B200_BM=bm4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj4_0 -s 1 -c 1 -o gpurun_out/prof/arap8192_jtj4 python scripts/exp/one_apply.py arap_warp 8192 > gpurun_out/prof/a.log 2>&1
MO_B200_JTJ=gather timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj_0 -s 1 -c 1 -o gpurun_out/prof/poisson8192_jtj python scripts/exp/one_apply.py poisson 8192 > gpurun_out/prof/c.log 2>&1
for f in gpurun_out/prof/*.log; do tail -n 3 $f; done
