"""GPU parity of NEXT-4 (int32 segments, exact clipping) through the C ABI
vs the exact-rational oracle (oracle/int_oracle.py): every output plane and flag bit-exact."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import int_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SCREEN = ([0, 0], [synth.INT_SCREEN - 1, synth.INT_SCREEN - 1])


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def run(torch, cs, planes, n, lo, hi):
    out, flags = cs.clip_int(torch.from_numpy(planes).cuda(), n, lo, hi)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:, :n], flags.cpu().numpy()[:n]


def check(torch, cs, planes, n, lo, hi):
    out, flags = run(torch, cs, planes, n, lo, hi)
    wout, wflags = O.clip_segments_i32(planes, n, lo, hi)
    bad = np.nonzero(flags != wflags)[0]
    assert bad.size == 0, (bad[:10], planes[:, bad[:3]])
    bad = np.nonzero((out != wout).any(axis=0))[0]
    assert bad.size == 0, (bad[:10], planes[:, bad[:3]], out[:, bad[:3]], wout[:, bad[:3]])
    return flags


def test_golden(torch, cs):
    cases = json.load(open(os.path.join(HERE, "golden", "int_examples.json")))["cases"]
    for c in cases:
        planes = np.zeros((4, 32), dtype=np.int32)
        planes[:, 0] = c["p"]
        w = c["win"]
        out, flags = run(torch, cs, planes, 1, w[:2], w[2:])
        assert flags[0] == c["flag"], c["id"]
        if c["flag"] == 1:
            assert out[:, 0].tolist() == c["q"], c["id"]
        else:
            assert (out[:, 0] == O.FILL).all(), c["id"]


@pytest.mark.parametrize("n", [1, 3, 4, 5, 31, 1023, 4097, 30001])
@pytest.mark.parametrize("mix", ["screen", "edge", "wide", "range", "mixed"])
def test_parity(torch, cs, n, mix):
    planes = synth.int_segments_host(1000 + n, n, mix)
    flags = check(torch, cs, planes, n, *SCREEN)
    if n > 1000 and mix in ("screen", "edge", "mixed"):
        assert (flags == 1).any() and (flags == 0).any()
        if mix == "range":
            assert (flags == 2).any()


def test_windows(torch, cs):
    B = 1 << 30
    planes = synth.int_segments_host(7, 20000, "wide")
    for lo, hi in (([-B, -B], [B, B]), ([5, 5], [5, 5]), ([-B, 0], [0, B]), ([-1000, -7], [123456, 999999])):
        check(torch, cs, planes, 20000, lo, hi)
    k = 1 << 14  # windows at and just past the 32-bit path's bound
    planes = synth.int_segments_host(8, 20000, "mixed")
    for lo, hi in (([-k, -k], [k, k]), ([-k - 1, 0], [k, k]), ([0, 0], [k + 1, 5]), ([-k, -k], [-k, -k])):
        check(torch, cs, planes, 20000, lo, hi)


def test_in_place_and_empty(torch, cs):
    n = 5000
    planes = synth.int_segments_host(3, n, "screen")
    wout, wflags = O.clip_segments_i32(planes, n, *SCREEN)
    t = torch.from_numpy(planes).cuda()
    out, flags = cs.clip_int(t, n, *SCREEN, out=t)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy()[:, :n], wout)
    assert np.array_equal(flags.cpu().numpy()[:n], wflags)
    cs.clip_int(t, 0, *SCREEN)  # n == 0: CLIP_OK, no launch


@pytest.mark.slow
def test_fullsize_sampled(torch, cs):
    """1e8 segments (the bench's next4 size, screen mix) checked on 4098 sampled rows,
    including the first and the last."""
    n = 100_000_000
    planes = synth.int_segments_host(77, n, "screen")
    out, flags = run(torch, cs, planes, n, *SCREEN)
    idx = np.random.default_rng(1).choice(n, 4096, replace=False)
    idx = np.concatenate([idx, [0, n - 1]])
    wout, wflags = O.clip_segments_i32(planes, n, *SCREEN, idx=idx)
    assert np.array_equal(flags[idx], wflags)
    assert np.array_equal(out[:, idx], wout)


# ---- the compacting int32 clip (NEXT-4 widening): visible rows in input order, flags 0/1/2 ----
def check_compact(torch, cs, planes, n, lo, hi, index_base=0):
    wout, wflags = O.clip_segments_i32(planes, n, lo, hi)
    vis = np.nonzero(wflags == 1)[0]
    b = cs.clip_int_compact(torch.from_numpy(planes).cuda(), n, lo, hi, with_index=True, with_flags=True,
                            index_base=index_base)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert cnt == len(vis)
    flags = b.flags.cpu().numpy()[:n]
    bad = np.nonzero(flags != wflags)[0]
    assert bad.size == 0, (bad[:10], flags[bad[:10]], wflags[bad[:10]], planes[:, bad[:3]])
    assert np.array_equal(b.index.cpu().numpy()[:cnt], vis + index_base)
    got = b.out.cpu().numpy()[:, :cnt]
    bad = np.nonzero((got != wout[:, vis]).any(axis=0))[0]
    assert bad.size == 0, (bad[:10], planes[:, vis[bad[:3]]], got[:, bad[:3]], wout[:, vis[bad[:3]]])
    assert not b.ws.any().item(), "workspace not left zero-filled"
    return flags


@pytest.mark.parametrize("n", [1, 5, 255, 256, 257, 3839, 3840, 3841, 30001, 200003])
@pytest.mark.parametrize("mix", ["screen", "edge", "wide", "range", "mixed"])
def test_compact_parity(torch, cs, n, mix):
    planes = synth.int_segments_host(2000 + n, n, mix)
    flags = check_compact(torch, cs, planes, n, *SCREEN, index_base=7)
    if n > 1000 and mix == "range":
        assert (flags == 2).any()


def test_compact_windows(torch, cs):
    B = 1 << 30
    k = 1 << 14
    planes = synth.int_segments_host(17, 50000, "mixed")
    for lo, hi in (([-B, -B], [B, B]), ([5, 5], [5, 5]), ([-k, -k], [k, k]), ([-k - 1, 0], [k, k]),
                   ([-1000, -7], [123456, 999999])):
        check_compact(torch, cs, planes, 50000, lo, hi)


def test_compact_empty_and_none_visible(torch, cs):
    planes = synth.int_segments_host(5, 4096, "screen")
    b = cs.clip_int_compact(torch.from_numpy(planes).cuda(), 0, *SCREEN)
    torch.cuda.synchronize()
    assert int(b.count.item()) == 0
    far = np.full((4, 4096), 1 << 20, dtype=np.int32)  # every segment beyond the window
    check_compact(torch, cs, far, 4000, *SCREEN)
