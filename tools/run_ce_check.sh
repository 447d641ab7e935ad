timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ieee or compress" > gpurun_out/ce1_tests.log 2>&1; tail -2 gpurun_out/ce1_tests.log
bash tools/quick_bench.sh ce1
timeout 300 python tools/spike_probe.py gpt2_xl 40 > gpurun_out/ce1_sp_gpt.txt 2>&1; head -3 gpurun_out/ce1_sp_gpt.txt
LOWDIFF_LIB=$PWD/tools/variants/m1smem/liblowdiff.so timeout 300 python tools/spike_probe.py gpt2_xl 40 > gpurun_out/ce1_sp_gpt_m1smem.txt 2>&1; head -1 gpurun_out/ce1_sp_gpt_m1smem.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^count_emit -s 20 -c 1 -o gpurun_out/ce1_prof_count_emit python bench.py --steps 4 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-c4-shape --no-recovery --no-update > /dev/null 2>&1
