# compute-sanitizer over the late round-2 kernels: jtj9t (2-row boxes, mask
# prefetch, evict_first), active tile / group lists, overlapped strip apply,
# peer reductions (LocalComm, opt-in)
mkdir -p gpurun_out/san2
MO_B200_JTJ=lct timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "golden_case and fma and cfg_" > gpurun_out/san2/memcheck_lct.txt 2>&1; echo "memcheck lct rc=$?"; tail -2 gpurun_out/san2/memcheck_lct.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_api_gpu.py -m gpu -q -p no:cacheprovider -k "rebound" > gpurun_out/san2/memcheck_lists.txt 2>&1; echo "memcheck lists rc=$?"; tail -2 gpurun_out/san2/memcheck_lists.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_shard_gpu.py -m gpu -q -p no:cacheprovider -k "overlapped and (lct or gather or ws) or peer_reductions" > gpurun_out/san2/memcheck_strips.txt 2>&1; echo "memcheck strips rc=$?"; tail -2 gpurun_out/san2/memcheck_strips.txt
MO_B200_JTJ=lct timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/exp/fe_sfs.py cfg_arap_warp_f32 > gpurun_out/san2/racecheck_lct.txt 2>&1; echo "racecheck lct rc=$?"; tail -2 gpurun_out/san2/racecheck_lct.txt
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "golden_case and fma and cfg_poisson" > gpurun_out/san2/initcheck_poisson.txt 2>&1; echo "initcheck rc=$?"; tail -2 gpurun_out/san2/initcheck_poisson.txt
