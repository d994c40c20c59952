#!/bin/bash
# One GPU-box pass: smoke, GPU parity tests, bench line, ncu launch list, ncu full capture of the commit kernel.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag] [what]
TAG=${1:-r01}
WHAT=${2:-all}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
if [[ $WHAT == all || $WHAT == test ]]; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
  head -c 600 gpurun_out/bench_$TAG.json; echo
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_commit_leaf} -s ${KSKIP:-3} -c 2 \
     -f -o gpurun_out/full_$TAG python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
