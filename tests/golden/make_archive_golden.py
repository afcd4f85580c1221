"""Golden archive digests of the reference's built-in setups (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_archive_golden.py

Runs ``mblight.create_solver("fdtd-reg-cayley", *mblight.builtin_setup(name))``
-- the reference's own solver through its own registry -- writes the result
with the reference's ``write_archive`` (writer_raw.py:40-92) and stores the
SHA-256 of every archive file in ``tests/golden/archives.json``.  The GPU test
(``tests/test_gpu_archive.py``) writes the GPU solver's archive of the same
setup and compares digests: "archive bytes identical", the contract of
pkg/tests/test_acceptance.py:279-312.  (The archives themselves are tens of
MB; the digests are what travels.)
"""

import hashlib
import json
import os
import sys
import time
from pathlib import Path
from tempfile import TemporaryDirectory

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import mblight  # noqa: E402

# (setup, gridpoints, end_time, stepper): the built-in defaults except where
# a shorter window keeps the reference run to seconds
SETUPS = {
    "ziolkowski1995": ("ziolkowski1995", None, None, "fdtd-reg-cayley"),
    "ziolkowski1995_rk4_60fs": ("ziolkowski1995", 4096, 60e-15, "fdtd-rk4"),
    "song2005": ("song2005", None, None, "fdtd-reg-cayley"),
}


def digest(folder: Path) -> dict:
    return {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(folder.iterdir())}


def main():
    out = {}
    threads = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 1))
    for key, (name, gridpoints, end_time, solver_name) in SETUPS.items():
        mblight.clear_material_library()
        dev, sce = mblight.builtin_setup(name, gridpoints=gridpoints, end_time=end_time)
        t = time.perf_counter()
        results = mblight.create_solver(solver_name, dev, sce, threads=threads).run()
        elapsed = time.perf_counter() - t
        with TemporaryDirectory() as tmp:
            mblight.write_archive(Path(tmp) / key, results, dev, sce)
            out[key] = {"setup": name, "gridpoints": gridpoints, "end_time": end_time, "solver": solver_name,
                        "files": digest(Path(tmp) / key), "elapsed_s": elapsed}
        print(f"{key}: {len(out[key]['files'])} files, {elapsed:.1f} s", flush=True)
    (HERE / "archives.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
