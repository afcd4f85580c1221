#!/bin/bash
# A/B timing of two builds of libmbgpu.so on the same box:
#   tools/ab.sh <dirA> <dirB> <rounds> <prof_step args...>
A=$1; B=$2; R=$3; shift 3
for i in $(seq 1 $R); do
  for v in $A $B; do
    echo -n "$v: "; MBGPU_LIB=$v/libmbgpu.so timeout 120 python tools/prof_step.py "$@" | grep -o "device.*"
  done
done
