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
  # one C2 step (tools/prof_step.py brackets it with cudaProfilerStart/Stop)
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu list rc=$?"
  IFS=',' read -ra KS <<< "${KREGEX:-k_commit_leaf}"
  for k in "${KS[@]}"; do
    timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 \
       -f -o gpurun_out/full_${TAG}_$k python tools/prof_step.py > gpurun_out/ncu_full_${TAG}_$k.log 2>&1; echo "ncu full $k rc=$?"
  done
fi
