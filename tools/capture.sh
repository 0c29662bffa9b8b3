#!/bin/bash
# Evidence for one config on the GPU box: bench line, ncu launch list and one
# `ncu --set full` capture of the dominant kernel (each ncu run only after the
# plain run exited 0).  Usage: tools/capture.sh <config> <kernel-regex> <tag>
# Outputs under gpurun_out/<tag>_*.
set -u
cfg=$1; kre=$2; tag=$3
mkdir -p gpurun_out
python bench.py --config "$cfg" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --config "$cfg" --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_l.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 1 -c 1 \
    -o gpurun_out/${tag}_full python bench.py --config "$cfg" --steps 1 --warmup 1 \
    --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
