"""paper_1110_5450_b200 — B200-native (sm_100a) batched line-segment clipping.

The data-parallel hot path BASELINE.json's north star assigns to arXiv 1110.5450:
outcode classification with trivial accept/reject, the window-edge-coordinate
intersection, clipped endpoints + visible flags, a stable one-pass compacting variant,
and a sharded multi-GPU mode that exchanges only per-shard visible counts.  See
DESIGN.md.  The compute lives in lib/libclipseg.so (C ABI: include/clipseg.h);
``clipseg`` is its thin binding and ``shard`` the torch.distributed plumbing.
"""
from . import clipseg  # noqa: F401  (raises if the native library is missing)

__all__ = ["clipseg"]
