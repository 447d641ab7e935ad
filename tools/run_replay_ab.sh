# replay A/B (not product): tools/run_replay_ab.sh TAG v1 v2 ... ("default" = in-tree build)
TAG=$1; shift
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/tools/variants/$v/liblowdiff.so; fi
  echo "$v $(timeout 300 python tools/replay_probe.py 100 1 2>&1 | tail -1)" >> gpurun_out/rab_$TAG.txt
  echo "$v $(timeout 300 python tools/replay_probe.py 100 8 2>&1 | tail -1)" >> gpurun_out/rab_$TAG.txt
done; done
