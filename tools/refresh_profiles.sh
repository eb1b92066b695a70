#!/bin/bash
# One GPU call (under gpurun) that regenerates the round's measured artifacts into
# gpurun_out/prof/: bench lines (ours: config 4 with e2e + CPU baseline, config 5; the
# reference arm), the config-4 launch list with DRAM bytes, and ncu --set full captures of
# the top K4 kernels.  Summaries are made locally afterwards (tools/*.py).
set -u
R=${1:-r01}
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/${R}_bench.log 2>&1
timeout 400 python bench.py --impl reference > $O/${R}_bench_reference.log 2>&1
timeout 400 python bench.py --config config5 --no-e2e --no-cpu-baseline --steps 3 > $O/${R}_bench_config5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_list.log 2>&1
for k in "ola_small_kernel<.int.512>" "ola_ip_kernel<.int.1024>" "ola_ip_kernel<.int.2048>" "mix_kernel" "rir_synth_kernel<.int.512, .int.4>"; do
  n=$(echo "$k" | tr -dc "a-z0-9_")
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" \
    --launch-skip 2 -c 1 -o $O/${R}_full_$n python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_$n.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:ola_ip_kernel<.int.16384>" \
  --launch-skip 2 -c 1 -o $O/${R}_full_ip16384_config5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config config5 > $O/ncu_ip16384.log 2>&1
ls -la $O
