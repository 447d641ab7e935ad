#!/bin/bash
# windowed-digit check (not product): compress parity + steady state, timings, merge TMA A/B
OUT=gpurun_out; TAG=${1:-win}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steady_state.py -q -x -k "compress or steady or resnet or gpt2 or bert" > $OUT/${TAG}_tests.log 2>&1; tail -n 3 $OUT/${TAG}_tests.log
timeout 300 python tools/spike_probe.py resnet50 200 > $OUT/${TAG}_sp_res.txt 2>&1
timeout 300 python tools/spike_probe.py gpt2_xl 60 > $OUT/${TAG}_sp_gpt.txt 2>&1
bash tools/quick_bench.sh $TAG
LOWDIFF_LIB=$PWD/tools/variants/mtma/liblowdiff.so timeout 300 python tools/spike_probe.py gpt2_xl 40 > $OUT/${TAG}_sp_gpt_tma.txt 2>&1
