"""Per-item timeline of the persistent two-level kernel (debug build aid).

    MBG_WAVE_TRACE=/tmp/t.bin python tools/prof_step.py cfg2 --steps 2048 --no-warm
    python tools/wave_trace.py /tmp/t.bin

Each work item logs {claimed, dependencies met, done, sm | cta << 32} in ns
(globaltimer); prints where the CTAs' time goes.
"""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
n_chunks, tiles = int(raw[0]), int(raw[1])
t = raw[2:].reshape(-1, 4).astype(np.int64)
claim, met, done = t[:, 0], t[:, 1], t[:, 2]
cta = (t[:, 3] >> 32).astype(np.int64)
t0 = claim.min()
span = done.max() - t0
wait = met - claim
work = done - met
order = np.lexsort((claim, cta))
c_sorted, cl, dn = cta[order], claim[order], done[order]
same = c_sorted[1:] == c_sorted[:-1]
gap = (cl[1:] - dn[:-1])[same]  # end of one item -> claim of the CTA's next one
n_cta = len(np.unique(cta))
busy = work.sum() / (n_cta * span)
print(f"chunks {n_chunks} items/chunk {tiles} CTAs {n_cta} span {span / 1e6:.3f} ms")
print(f"work/item  median {np.median(work) / 1e3:.1f} us  p99 {np.percentile(work, 99) / 1e3:.1f} us  max {work.max() / 1e3:.1f}")
print(f"wait/item  median {np.median(wait) / 1e3:.2f} us  mean {wait.mean() / 1e3:.2f}  p99 {np.percentile(wait, 99) / 1e3:.2f}"
      f"  total share {wait.sum() / (n_cta * span):.3%}")
print(f"gap (done->next claim) median {np.median(gap) / 1e3:.2f} us  mean {gap.mean() / 1e3:.2f}"
      f"  share {gap.sum() / (n_cta * span):.3%}")
print(f"work share of CTA time {busy:.3%}")
start = np.sort(claim - t0)[: n_cta]
print(f"ramp: last CTA starts at {start[-1] / 1e3:.1f} us; tail: first CTA idle at "
      f"{(np.sort(np.bincount(cta, weights=None) * 0)[0])}")
ends = np.array([dn[c_sorted == c].max() for c in np.unique(cta)]) - t0
print(f"tail: CTA finish times min {ends.min() / 1e6:.3f} ms  max {ends.max() / 1e6:.3f} ms")
wt = work.reshape(n_chunks, tiles)
print("slowest item kinds (work us):", np.round(np.sort(wt.mean(axis=0))[-8:] / 1e3, 1))
