mkdir -p gpurun_out/san
for v in ws lc; do
MO_B200_JTJ=$v MO_B200_BM=bm8 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "golden_case and fma and cfg_" > gpurun_out/san/memcheck_$v.txt 2>&1; echo "memcheck $v rc=$?"; tail -3 gpurun_out/san/memcheck_$v.txt
done
MO_B200_JTJ=lc MO_B200_BM=bm8 timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/exp/fe_sfs.py cfg_arap_warp_f32 > gpurun_out/san/racecheck_lc.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san/racecheck_lc.txt
MO_B200_JTJ=ws MO_B200_BM=bm8 timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/exp/fe_sfs.py cfg_poisson_f32 > gpurun_out/san/racecheck_ws.txt 2>&1; echo "racecheck ws rc=$?"; tail -3 gpurun_out/san/racecheck_ws.txt
MO_B200_DEFER=1 timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "pcg_schemes and deferred and cfg_" > gpurun_out/san/initcheck_defer.txt 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/san/initcheck_defer.txt
