#!/bin/bash
# One GPU call (under gpurun) that regenerates the round's measured artifacts into
# gpurun_out/prof/: bench lines (ours: config 4 with e2e + CPU baseline + parity, configs 2 / 3 / 5,
# the strong-scaling per-rank share at N = 8; the reference arm), the config-4 launch list with
# DRAM bytes, and ncu --set full captures of the top kernels.  Summaries are made locally
# afterwards (tools/launch_summary.py, tools/k4_traffic.py, tools/ncu_summary.py).
set -u
R=${1:-r02}
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/${R}_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/${R}_bench_reference.log 2>&1; echo "reference rc=$?"
for c in config2 config3 config5; do
  timeout 600 python bench.py --config $c --no-e2e --steps 3 > $O/${R}_bench_$c.log 2>&1; echo "$c rc=$?"
done
timeout 600 python bench.py --utterances 512 --no-cpu-baseline > $O/${R}_bench_strong512.log 2>&1; echo "512 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/${R}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown > $O/ncu_list.log 2>&1
echo "launch list rc=$?"
for k in "ola_ipc_kernel<.int.4096>" "ola_ipc_kernel<.int.8192>" \
         "rir_synth_kernel<.int.128, .int.4" "rir_bound_kernel<.int.512"; do
  n=$(echo "$k" | tr -dc "a-z0-9_")
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" \
    --launch-skip 2 -c 1 -o $O/${R}_full_$n python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > $O/ncu_$n.log 2>&1
  echo "$n rc=$?"
  # the copy-back limit is 64 MiB: raw metrics as CSV for every capture, the report itself
  # only for the two largest K4 kernels
  ncu -i $O/${R}_full_$n.ncu-rep --page raw --csv > $O/${R}_full_${n}_raw.csv 2>/dev/null
  ncu -i $O/${R}_full_$n.ncu-rep --page source --csv > $O/${R}_full_${n}_source.csv 2>/dev/null
  case $n in ola_ipc_kernelint4096) ;; *) rm -f $O/${R}_full_$n.ncu-rep ;; esac
done
# the reference's block sizes executed as planned (RSG_REBLOCK=0): the pre-re-blocking K4 mix
RSG_REBLOCK=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/${R}_bench_reblock_off.log 2>&1; echo "reblock-off rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:ola_ip_kernel<.int.16384>" \
  --launch-skip 2 -c 1 -o $O/${R}_full_ip16384_config5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown --config config5 > $O/ncu_ip16384.log 2>&1
echo "ip16384 rc=$?"
ncu -i $O/${R}_full_ip16384_config5.ncu-rep --page raw --csv > $O/${R}_full_ip16384_config5_raw.csv 2>/dev/null
rm -f $O/${R}_full_ip16384_config5.ncu-rep
du -sh $O
ls -la $O
