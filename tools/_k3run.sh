timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_balance.py tests/test_gpu_edges.py -x -q 2>&1 | tail -3
python tools/bench_configs.py --configs 4 --steps 2 | cut -c1-400
bash tools/k3_ipb.sh
