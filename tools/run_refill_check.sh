#!/bin/bash
# compress parity (incl. steady state) + spike probe + quick bench lines after a compress change
OUT=gpurun_out; TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steady_state.py -q -x -k "compress or steady or resnet or gpt2 or bert" > $OUT/${TAG}_tests.log 2>&1; tail -n 3 $OUT/${TAG}_tests.log
timeout 300 python tools/spike_probe.py resnet50 200 > $OUT/${TAG}_sp_res.txt 2>&1
timeout 300 python tools/spike_probe.py gpt2_xl 60 > $OUT/${TAG}_sp_gpt.txt 2>&1
bash tools/quick_bench.sh $TAG
