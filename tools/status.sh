#!/bin/bash
# Reproduce the cell-update rates of DESIGN.md section 8 on one B200 (about 2 minutes):
#   bash tools/status.sh
set -e
cd "$(dirname "$0")/.."
run() { echo -n "$*: "; timeout 300 python tools/prof_step.py "$@" | grep -o "device.*"; }
run cfg1 --steps 26196                      # two-level SIT, 32768 cells, the full run (one launch per chunk)
run cfg2 --steps 20000                      # two-level, 2^22 cells, the full 20000-step run (persistent kernel)
run cfg3 --steps 96                         # three-level Lambda medium, 2^23 cells (real-operator path)
run cfg4 --steps 96                         # six-level QCL-like medium, 2^24 cells (complex Hamiltonian)
run cfg4 --real --steps 96                  # its real-Hamiltonian twin
run cfg2 --stepper rk4 --steps 48           # RK4 on the same media
run cfg3 --stepper rk4 --steps 48
run cfg4 --stepper rk4 --steps 48
timeout 300 python tools/slab_step.py --config cfg2 --world 3 | tail -1          # slab path, per rank
timeout 300 python tools/slab_step.py --config cfg5 --world 3 --period 16 --tile-steps 4 --steps 512 | tail -1
timeout 600 python tools/points_bench.py --systems 4096 | tail -1                 # batched single points
timeout 600 python tools/points_bench.py --systems 4096 --sweep media | tail -1   # 4096 distinct media
timeout 600 python tools/published_setups.py 2>/dev/null                          # the paper's examples, public call
timeout 600 python tools/small_nlevel.py 2>/dev/null                              # small N-level domains
