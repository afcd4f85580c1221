#!/bin/bash
# Timing of tuning builds (_var/<name>/libmbgpu.so) on the same box:
#   tools/var_sweep.sh "<prof_step args>" name1 name2 ...   (name "cur" = the in-tree build)
ARGS=$1; shift
for v in "$@"; do
  if [ "$v" = cur ]; then lib=paper_2005_05412_b200/_build/libmbgpu.so; else lib=_var/$v/libmbgpu.so; fi
  for r in 1 2; do
    echo -n "$v [$ARGS]: "; MBGPU_LIB=$lib timeout 120 python tools/prof_step.py $ARGS | grep -o "device.*"
  done
done
