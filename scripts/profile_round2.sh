#!/bin/bash
# Round-2 GPU evidence (run under gpurun from the repo root): bench line per
# config, ncu launch list of one timed solve per large config (kernels forced
# to the bench's choice, final solve only), one `ncu --set full` capture of
# each headline kernel.  profiles/summarize.py turns gpurun_out/r02f into profiles/.
O=gpurun_out/r02f
mkdir -p $O
for a in "arap_warp_8192|" "arap_warp_1024|--size 1024" "poisson_8192|--config poisson --size 8192" "poisson_512|--config poisson" "sfs|--config sfs" "arap_mesh|--config arap_mesh"; do
  tag=${a%%|*}; args=${a#*|}
  extra=--no-cpu-baseline; [ "$tag" = arap_warp_8192 ] && extra=
  timeout 900 python bench.py $args $extra > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$tag rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
L() { tag=$1; cfg=$2; shift 2; env MO_B200_NOGRAPH=1 "$@" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ll_$tag.csv python scripts/exp/one_solve.py $cfg > $O/ll_$tag.log 2>&1; grep LAUNCHES $O/ll_$tag.log; }
L arap_warp_8192 "arap_warp 8192" MO_B200_JTJ=lct MO_B200_BM=bm8
L poisson_8192 "poisson 8192" MO_B200_JTJ=gather MO_B200_BM=prog
L arap_warp_1024 "arap_warp 1024" MO_B200_JTJ=lct MO_B200_BM=bm8
F() { tag=$1; k=$2; s=$3; shift 3; env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o $O/$tag python scripts/exp/one_solve.py $CFG > $O/ncu_$tag.log 2>&1; tail -1 $O/ncu_$tag.log; }
CFG="arap_warp 8192" F arap8192_jtj9t mo_gather_jtj9t_0 30 MO_B200_JTJ=lct MO_B200_BM=bm8
CFG="arap_warp 8192" F arap8192_bm8c mo_gather_bm8c_0 1 MO_B200_JTJ=lct MO_B200_BM=bm8
CFG="arap_warp 8192" F arap8192_dp k_pcg_dp 3 MO_B200_JTJ=lct MO_B200_BM=bm8
CFG="poisson 8192" F poisson8192_jtj mo_gather_jtj_0 30 MO_B200_JTJ=gather MO_B200_BM=prog
CFG="poisson 8192" F poisson8192_bm mo_gather_bm_0 1 MO_B200_JTJ=gather MO_B200_BM=prog
ls $O
