mkdir -p gpurun_out; rm -f gpurun_out/p_*.json
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/p_first4096.json 2>/dev/null
RSG_FIRST_CHUNK=0 $B > gpurun_out/p_nofirst.json 2>/dev/null
RSG_FIRST_CHUNK=2048 $B > gpurun_out/p_first2048.json 2>/dev/null
RSG_FIRST_CHUNK=8192 $B > gpurun_out/p_first8192.json 2>/dev/null
RSG_FIRST_CHUNK=4096 RSG_CHUNK_PAIRS=16384 $B > gpurun_out/p_c16384.json 2>/dev/null
RSG_TRACE=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/trace.json 2> gpurun_out/trace.err
python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
