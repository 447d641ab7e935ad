# replay ncu capture (not product): one 10-step GPT-2 XL Adam replay kernel, full set + source
# tools/run_replay_ncu.sh TAG [WORLD]
set -u
O=gpurun_out/rncu_${1:-x}
W=${2:-1}
mkdir -p $O
timeout 300 python tools/replay_probe.py 100 $W > $O/time.txt 2>&1; cat $O/time.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o $O/replay python tools/replay_probe.py 10 $W > $O/ncu.log 2>&1; tail -n 2 $O/ncu.log
