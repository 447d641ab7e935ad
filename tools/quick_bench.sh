#!/bin/bash
# quick A/B of the compress chain on the GPU box: GPT-2 XL and ResNet-50 bench lines (no side legs)
# usage: tools/quick_bench.sh TAG   -> gpurun_out/qb_TAG_{gpt,res}.json
TAG=${1:-x}
OPTS="--no-recovery --no-writer --no-replica --no-snapshot --no-union --no-cpu --no-full --no-update --no-e2e --no-c4-shape"
timeout 200 python bench.py --steps 20 --warmup 20 $OPTS > gpurun_out/qb_${TAG}_gpt.json 2> gpurun_out/qb_${TAG}_gpt.err
timeout 200 python bench.py --workload resnet50 --steps 200 --warmup 20 $OPTS > gpurun_out/qb_${TAG}_res.json 2> gpurun_out/qb_${TAG}_res.err
