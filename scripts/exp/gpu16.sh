# jtj9t at 8192^2: unperturbed time and one full ncu capture
O=gpurun_out/g16; mkdir -p $O
timeout 300 env MO_B200_JTJ=lct MO_B200_BM=bm8 python scripts/exp/ktime.py arap_warp 8192 2>&1 | grep '^{'
timeout 600 env MO_B200_JTJ=lct MO_B200_BM=bm8 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj9t_0 -s 3 -c 1 -o $O/jtj9t python scripts/exp/one_apply.py arap_warp 8192 6 > $O/ncu.log 2>&1; tail -2 $O/ncu.log
