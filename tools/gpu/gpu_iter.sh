#!/bin/bash
# usage: tools/gpu/gpu_iter.sh TAG [pytest-args]   (runs on the GPU box)
TAG=$1; shift
mkdir -p gpurun_out
if [ "$1" != "nobench" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
fi
timeout 300 python bench.py --steps 20 --warmup 5 --profile > gpurun_out/bench$TAG.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench$TAG.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches$TAG.csv | tail -15
