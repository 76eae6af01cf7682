mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02/gputest.log 2>&1; echo tests_rc=$?
tail -4 gpurun_out/r02/gputest.log
for a in "arap_warp_8192|" "arap_warp_1024|--size 1024" "poisson_8192|--config poisson --size 8192" "poisson_512|--config poisson" "sfs|--config sfs" "arap_mesh|--config arap_mesh"; do
  tag=${a%%|*}; args=${a#*|}
  timeout 900 python bench.py $args --no-cpu-baseline > gpurun_out/r02/bench_$tag.json 2> gpurun_out/r02/bench_$tag.err; echo "$tag rc=$?"
done
MO_B200_JTJ=lc timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj9_0 -s 1 -c 1 -o gpurun_out/r02/arap8192_jtj9 python scripts/exp/one_apply.py arap_warp 8192 > gpurun_out/r02/ncu_a.log 2>&1
MO_B200_JTJ=gather timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj_0 -s 1 -c 1 -o gpurun_out/r02/poisson8192_jtj python scripts/exp/one_apply.py poisson 8192 > gpurun_out/r02/ncu_b.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pcg_dp -s 3 -c 1 -o gpurun_out/r02/arap8192_dp python scripts/exp/one_solve.py arap_warp 8192 > gpurun_out/r02/ncu_c.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pcg_update_r -s 3 -c 1 -o gpurun_out/r02/arap8192_upd python scripts/exp/one_solve.py arap_warp 8192 > gpurun_out/r02/ncu_d.log 2>&1
MO_B200_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02/ll_poisson8192.csv python scripts/exp/one_solve.py poisson 8192 > /dev/null 2>&1
ls gpurun_out/r02
