# bench lines only (not product): default line + C2/C3/C4-sweep configs, no profilers
set -u
mkdir -p gpurun_out/r2
timeout 900 python bench.py --steps 20 --warmup 8 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; tail -n 2 gpurun_out/p_bench.err
timeout 1500 bash tools/run_configs.sh
