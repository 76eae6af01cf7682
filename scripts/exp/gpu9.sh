mkdir -p gpurun_out/r02
L() { tag=$1; shift; env MO_B200_NOGRAPH=1 "$@" timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/ll_$tag.csv python scripts/exp/one_solve.py ${CFG} > gpurun_out/r02/ll_$tag.log 2>&1; grep LAUNCHES gpurun_out/r02/ll_$tag.log; }
CFG="arap_warp 1024" L arap1024_defer MO_B200_JTJ=lc MO_B200_BM=bm8
CFG="arap_warp 1024" L arap1024_nodefer MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_NO_DEFER=1
CFG="poisson 512" L poisson512_defer MO_B200_JTJ=gather MO_B200_BM=prog
CFG="poisson 512" L poisson512_nodefer MO_B200_JTJ=gather MO_B200_BM=prog MO_B200_NO_DEFER=1
CFG="arap_warp 8192" L arap8192 MO_B200_JTJ=lc MO_B200_BM=bm8
CFG="poisson 8192" L poisson8192 MO_B200_JTJ=gather MO_B200_BM=prog
