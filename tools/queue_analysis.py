"""Queue-state analysis of a saved trace (tools/trace_report.py ... out.npy):
over time, how many CTAs sit in the pop loop while how many tasks are queued
(pushed, not yet claimed). Idle CTAs next to queued tasks = pop overhead;
busy CTAs next to a long queue = priority / capacity limit (development aid).

    python tools/queue_analysis.py trace.npy
"""
import sys

import numpy as np

tr = np.load(sys.argv[1])
t0 = tr["taken"].min()
taken = (tr["taken"] - t0) / 1e3
ready = (tr["ready"] - t0) / 1e3
done = (tr["done"] - t0) / 1e3
push = tr["c_store"].astype(np.float64)
has_push = push > 0
push = np.where(has_push, (push - t0) / 1e3, np.nan)
span = done.max()
grid = np.linspace(0, span, 41)[:-1]
print(f"span {span:.1f} us, {len(tr)} tasks, {has_push.sum()} queued through the ready queues")
print("  t(us)   popping  running  queued  (queued = pushed, not yet claimed)")
for t in grid:
    popping = ((taken <= t) & (ready > t)).sum()
    running = ((ready <= t) & (done > t)).sum()
    queued = (has_push & (push <= t) & (ready > t) & ~((taken <= t) & (ready > t))).sum()
    print(f"  {t:7.0f}  {popping:7d}  {running:7d}  {queued:6d}")
w = ready - taken
print(f"pop wait: mean {w.mean():.2f} us, p50 {np.median(w):.2f}, p90 {np.percentile(w, 90):.2f}, "
      f"max {w.max():.2f}")
q = (ready - push)[has_push]
print(f"push -> start: mean {np.nanmean(q):.1f} us, p50 {np.nanmedian(q):.1f}, p90 {np.nanpercentile(q, 90):.1f}")
