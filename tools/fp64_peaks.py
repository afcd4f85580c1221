"""FP64 FMA throughput of the device by operand pattern (TFLOP/s): the
roofline denominator of bench.py (two registers + a uniform addend, the pipe's
peak) against shared multiplier/addend registers, one shared multiplier
register, and three distinct register operands per DFMA."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2005_05412_b200 import native  # noqa: E402

lib = native.load()
v = C.c_double(0)
for _ in range(2):
    rc = lib.mbg_fp64_peak(0, C.byref(v))
print(f"mbg_fp64_peak (mode 1, the roofline denominator): rc={rc} {v.value:.2f} TFLOP/s")
for mode, what in ((1, "two registers + uniform addend"), (0, "multiplier and addend registers shared by every DFMA"),
                   (2, "one multiplier register shared by consecutive DFMAs"),
                   (3, "three distinct register operands")):
    for _ in range(2):
        rc = lib.mbg_fp64_peak_operands(0, mode, C.byref(v))
    print(f"mode {mode} ({what}): rc={rc} {v.value:.2f} TFLOP/s")
