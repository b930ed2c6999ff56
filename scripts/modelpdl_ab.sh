for v in 0 1 0 1; do echo "WS_MODELPDL=$v"; WS_MODELPDL=$v python scripts/graph_ab.py 2>&1 | head -2; WS_MODELPDL=$v python scripts/probe.py configs1 lbm15 | grep "n="; done
WS_MODELPDL=1 timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
