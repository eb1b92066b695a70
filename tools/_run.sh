mkdir -p gpurun_out; rm -f gpurun_out/p_*.json
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_blocks or every_fft or reference_blocking or render_config or boundaries" 2>&1 | tail -15
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/p_ipc.json 2>gpurun_out/p_ipc.err
RSG_IPC=0,0 $B > gpurun_out/p_noipc.json 2>/dev/null
RSG_IPC=12,12 $B > gpurun_out/p_ipc12.json 2>/dev/null
