mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_blocks or render_config or reference_blocking" 2>&1 | tail -3
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/p_k3.json 2>gpurun_out/p_k3.err
RSG_TRACE=1 python bench.py --config config5 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/trace5.json 2> gpurun_out/trace5.err
