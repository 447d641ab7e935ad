#!/bin/bash
# A/B of tuning variants (not product): compress-only per-call times (tools/spike_probe.py)
# usage: tools/run_ab.sh TAG v1 v2 ...   (variants under tools/variants/, "default" = in-tree build)
TAG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/tools/variants/$v/liblowdiff.so; fi
  echo "== $v (rep $rep)" >> gpurun_out/ab_$TAG.txt
  timeout 300 python tools/spike_probe.py resnet50 150 2>&1 | head -5 >> gpurun_out/ab_$TAG.txt
  timeout 300 python tools/spike_probe.py gpt2_xl 40 2>&1 | head -5 >> gpurun_out/ab_$TAG.txt
done
done
