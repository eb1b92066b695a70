mkdir -p gpurun_out; rm -f gpurun_out/t_*.json
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/t_base.json 2>/dev/null
RSG_HOST_THREADS=16 $B > gpurun_out/t_h16.json 2>/dev/null
RSG_HOST_THREADS=4 $B > gpurun_out/t_h4.json 2>/dev/null
RSG_HOST_THREADS=12 $B > gpurun_out/t_h12.json 2>/dev/null
nproc
