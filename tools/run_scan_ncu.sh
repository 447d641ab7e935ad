# scan ncu capture (not product): one steady-state scan_kernel (call 21) of the GPT-2 XL bench loop
set -u
O=gpurun_out/sncu_${1:-x}
mkdir -p $O
SHORT="python bench.py --steps 4 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-c4-shape --no-recovery --no-update --trace-calls 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^scan_kernel -s 20 -c 1 -o $O/scan $SHORT > $O/ncu.log 2>&1; tail -n 2 $O/ncu.log
