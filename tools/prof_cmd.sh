#!/usr/bin/env bash
# One ncu --set full capture (with source) of the k_win launch of a bench
# command, after the same command has exited 0 without ncu (B200_PROFILING.md).
# Usage (on the box): bash tools/prof_cmd.sh <tag> <bench args...>
set -u
TAG=$1; shift
OUT=gpurun_out/prof; mkdir -p $OUT
python bench.py --steps 10 --warmup 3 --no-cpu --no-alt "$@" > $OUT/$TAG.plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_win -s 5 -c 1 -o $OUT/$TAG -f \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-alt "$@" > $OUT/$TAG.ncu.log 2>&1
echo "$TAG rc=$?"
