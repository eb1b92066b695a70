mkdir -p gpurun_out; rm -f gpurun_out/p_*.json
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_blocks or render_config4" 2>&1 | tail -3
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/p_ipc_pred.json 2>gpurun_out/p_ipc.err
RSG_IPC_MINB=4 $B > gpurun_out/p_ipc_minb4.json 2>/dev/null
RSG_IPC_MINB=4 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_blocks" 2>&1 | tail -3
