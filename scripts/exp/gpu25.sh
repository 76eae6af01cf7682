export MO_B200_P2P_TIMEOUT_S=5
MO_B200_LOCAL_P2P=1 timeout 300 python scripts/exp/strip_p2p.py arap_warp 2048 4
MO_B200_LOCAL_P2P=1 timeout 300 python scripts/exp/strip_p2p.py poisson 2048 4
timeout 1200 python -m pytest tests/test_shard_gpu.py -m gpu -p no:cacheprovider -x -q 2>&1 | tail -3
