# Round-2 final profiling pass (not product): GPU tests, default bench line, config lines, ncu
# launch list and full captures of the top kernels -> gpurun_out/ (copied to profiles/ by hand)
set -u
SKIP_TESTS=0 bash tools/profile_r02.sh r02f
bash tools/run_configs.sh r02f
