#!/bin/bash
# On the GPU box: bench the built library, then rebuild with the given -D flags and bench again.
# usage: tools/variant_bench.sh <outdir> "<bench args>" "<-D flags|env:VAR=V>" ...
set -u
O=$1; shift
A=$1; shift
mkdir -p $O
python tools/fin_probe.py 1 2 2>&1 | grep seed
python bench.py $A > $O/base.log 2>&1; tail -1 $O/base.log | cut -c1-160
i=0
for F in "$@"; do
  i=$((i+1))
  echo "== $F"
  case "$F" in
    env:*) env "${F#env:}" python tools/fin_probe.py 1 2 2>&1 | grep seed; env "${F#env:}" python bench.py $A > $O/var_$i.log 2>&1; tail -1 $O/var_$i.log | cut -c1-160; continue;;
  esac
  touch paper_1712_03439_b200/csrc/mixfin.cuh
  make -s -j8 EXTRA="$F" paper_1712_03439_b200/_lib/libroomsim_gpu.so > $O/make_$i.log 2>&1 || { echo "build failed: $F"; tail -5 $O/make_$i.log; continue; }
  python tools/fin_probe.py 1 2 2>&1 | grep seed
  python bench.py $A > $O/var_$i.log 2>&1; tail -1 $O/var_$i.log | cut -c1-160
done
