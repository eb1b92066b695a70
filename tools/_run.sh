mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -x -q -k "truncation or invariance or rirs_bit_exact or render_config or rir_" 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:rir_synth|rir_bound" --csv --log-file gpurun_out/k1_new.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p_a.json 2>gpurun_out/p_a.err
