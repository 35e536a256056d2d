#!/usr/bin/env python3
"""Summarise GI_DEBUG_SEG_TIMING output: per-CTA busy time, staging time, chunks, units (last launch)."""
import sys
import numpy as np

rows = [list(map(int, l.split(","))) for l in open(sys.argv[1]) if l.strip()]
ctas = max(r[0] for r in rows) + 1
full = np.array(rows[-ctas:], dtype=np.float64)
last = full[:, :7]
t0 = last[:, 3].min()
start, end, stage, units = last[:, 3] - t0, last[:, 4] - t0, last[:, 5], last[:, 6]
pieces = last[:, 7] if last.shape[1] > 7 else np.zeros(len(last))
chunks = last[:, 2] - last[:, 1]
dur = end - start
print(f"kernel span {end.max() / 1e3:.1f} us; CTA busy mean {dur.mean() / 1e3:.1f} min {dur.min() / 1e3:.1f} "
      f"max {dur.max() / 1e3:.1f} us; start skew {start.max() / 1e3:.1f} us")
print(f"staging wait mean {stage.mean() / 1e3:.2f} max {stage.max() / 1e3:.2f} us; units/CTA mean {units.mean():.1f} "
      f"max {units.max():.0f}; chunks/CTA mean {chunks.mean():.0f} min {chunks.min():.0f} max {chunks.max():.0f}")
for q in [0, 10, 25, 50, 75, 100, 120, 140, ctas - 1]:
    if q < ctas:
        print(f"  cta {q:3d}: chunks {chunks[q]:6.0f} pieces/chunk {pieces[q] / max(chunks[q], 1):6.1f} units {units[q]:3.0f} busy {dur[q] / 1e3:6.1f} us "
              f"stage {stage[q] / 1e3:5.2f} us  ns/chunk {dur[q] / max(chunks[q], 1):6.1f}")

# least-squares fit: busy = a*chunks + b*pieces + c*units (ns)
X = np.stack([chunks, pieces, units], 1)
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
pred = X @ coef
print(f"fit busy ~ {coef[0]:.1f} ns/chunk + {coef[1]:.2f} ns/piece + {coef[2]:.0f} ns/unit; "
      f"rms err {np.sqrt(np.mean((pred - dur) ** 2)) / 1e3:.2f} us; balanced span ~ {dur.sum() / len(dur) / 1e3:.1f} us")

if full.shape[1] >= 11:  # + unstaged records, staged units, first and last unit per CTA
    order = np.argsort(-dur)[:8]
    print("slowest CTAs: cta busy_us records unstaged_records staged_units units[first..last]")
    for q in order:
        print(f"  {q:3d} {dur[q] / 1e3:7.1f} {chunks[q]:6.0f} {full[q, 7]:6.0f} {full[q, 8]:4.0f} [{full[q, 9]:.0f}..{full[q, 10]:.0f}]")
