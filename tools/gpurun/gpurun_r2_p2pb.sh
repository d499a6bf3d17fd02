# the separate-broadcast P2P path as a test
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_gpu_zero_p2p.py -q -k "separate_broadcast" 2>&1 | tail -2
