O=gpurun_out/r02g; mkdir -p $O
L() { tag=$1; cfg=$2; shift 2; env MO_B200_NOGRAPH=1 "$@" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ll_$tag.csv python scripts/exp/one_solve.py $cfg > $O/ll_$tag.log 2>&1; grep LAUNCHES $O/ll_$tag.log; }
L arap_warp_8192 "arap_warp 8192" MO_B200_JTJ=lct MO_B200_BM=bm8
L arap_warp_1024 "arap_warp 1024" MO_B200_JTJ=lct MO_B200_BM=bm8
