#!/bin/bash
# Bounds-checked build (every global access of the step, sample and halo
# kernels checked against its buffer's extent; a violation prints the site and
# traps -- see MBG_CHK in csrc/mbg_params.cuh) and the GPU test suite run
# against it.  compute-sanitizer is closed on this GPU pool; this is the
# memory-safety evidence in its place.
#   make -C paper_2005_05412_b200/csrc OUT=../../_var/bounds EXTRA=-DMBG_BOUNDS=1   (here, CPU)
#   tools/bounds_check.sh > profiles/<tag>_bounds_check.log                         (GPU box)
set -o pipefail
lib=_var/bounds/libmbgpu.so
test -f $lib || { echo "build $lib first"; exit 2; }
echo "library: $lib ($(stat -c %s $lib) bytes)"
MBGPU_LIB=$lib timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -25
rc=$?
echo "pytest rc=$rc"
MBGPU_LIB=$lib timeout 600 python tools/sanitize_cases.py 2>&1 | tail -20
echo "sanitize_cases rc=$?"
