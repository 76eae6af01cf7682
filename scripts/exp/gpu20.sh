O=gpurun_out/g20; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_bm8c_0 -s 1 -c 1 -o $O/bm8c python scripts/exp/one_apply.py arap_warp 8192 3 > $O/ncu1.log 2>&1; tail -1 $O/ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj9t_0 -s 3 -c 1 -o $O/jtj9t python scripts/exp/one_apply.py arap_warp 8192 6 > $O/ncu2.log 2>&1; tail -1 $O/ncu2.log
