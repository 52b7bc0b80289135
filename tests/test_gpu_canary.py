"""Out-of-bounds write detection for every C-ABI entry point (compute-sanitizer is not
available on the GPU pool): each output buffer is a view into a larger allocation whose
remainder holds a sentinel byte pattern, workspaces are passed at their exact documented
size, and after the call (checked against the oracle) every byte outside the documented
write set must still hold the sentinel — plane padding [n, ld) and rows >= count included
(include/clipseg.h: "kernels may read, never write, the padding"; "rows >= count are not
written").  Inputs must be unchanged."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

S = 0x5A          # sentinel byte
PAD = 64          # guard elements after every buffer / plane
UNIT = {2: ([0.0, 0.0], [1.0, 1.0]), 3: ([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])}


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


class Guarded:
    """rows x cols elements of `dtype` (rows = 0: 1-D) inside a sentinel-filled allocation
    with PAD guard elements after each row; `.t` is the view handed to the library."""

    def __init__(self, torch, rows, cols, dtype, device="cuda", pin=False):
        esz = torch.empty(0, dtype=dtype).element_size()
        r = max(rows, 1)
        self.raw = torch.full((r * (cols + PAD) * esz,), S, dtype=torch.uint8, device=device)
        if pin:
            self.raw = self.raw.pin_memory()
        full = self.raw.view(dtype).view(r, cols + PAD)
        self.t = full[:, :cols] if rows else full[0, :cols]
        self.rows, self.cols, self.esz = r, cols, esz

    def untouched_from(self, start):
        """True iff every byte of columns [start, cols + PAD) of every row is the sentinel."""
        b = self.raw.view(self.rows, (self.cols + PAD) * self.esz)[:, start * self.esz:]
        return bool((b == S).all().item())


class Bufs:
    pass


def compact_bufs(torch, cs, n, rows, dtype):
    b = Bufs()
    ld = cs.clip_plane_stride(n)
    b.g_out = Guarded(torch, rows, ld, dtype)
    b.g_idx = Guarded(torch, 0, max(n, 1), torch.int64)
    b.g_fl = Guarded(torch, 0, max(n, 1), torch.uint8)
    b.g_cnt = Guarded(torch, 0, 1, torch.int64)
    b.g_ws = Guarded(torch, 0, max(int(cs.clip_compact_workspace_bytes(n)), 1), torch.uint8)
    b.out, b.index, b.flags, b.count, b.ws = b.g_out.t, b.g_idx.t, b.g_fl.t, b.g_cnt.t, b.g_ws.t
    b.ws.zero_()  # the workspace contract: zero-filled before first use
    return b


def check_compact_guards(b, n, cnt):
    assert b.g_out.untouched_from(cnt), "compacted rows >= count or plane padding written"
    assert b.g_idx.untouched_from(cnt), "out_index past count written"
    assert b.g_fl.untouched_from(n), "flags past n written"
    assert b.g_cnt.untouched_from(1)
    assert b.g_ws.untouched_from(b.ws.numel()), "workspace overrun"
    assert not b.ws.any().item(), "workspace not left zero-filled for the next call"


@pytest.mark.parametrize("dim,dt,n", [(2, np.float32, 70001), (2, np.float64, 20011), (3, np.float32, 30011),
                                      (3, np.float64, 9001), (2, np.float32, 5), (2, np.float32, 0)])
def test_compact_guards(torch, cs, dim, dt, n):
    P, _ = synth.fill_host(synth.UNIFORM, dim, synth.seed_for(42), max(n, 1), dtype=dt)
    want, widx, wcnt, wfl = oracle.compact(P, n, *UNIT[dim], dim, index_base=5, with_flags=True)
    dP = torch.from_numpy(P).cuda()
    before = dP.clone()
    b = compact_bufs(torch, cs, n, 2 * dim, dP.dtype)
    cs.clip_compact(dP, n, *UNIT[dim], bufs=b, index_base=5)
    torch.cuda.synchronize()
    c = int(b.count.item())
    assert c == wcnt
    assert np.array_equal(b.flags.cpu().numpy()[:n], wfl[:n])
    assert np.array_equal(b.index.cpu().numpy()[:c], widx)
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :c]), bits(want[:, :c]))
    check_compact_guards(b, n, c)
    assert torch.equal(dP, before)


@pytest.mark.parametrize("fam,dim,dt,n", [(synth.ADVERSARIAL, 2, np.float32, 10007), (synth.UNIFORM, 3, np.float64, 4099),
                                          (synth.UNIFORM, 2, np.float32, 3)])
def test_dense_guards(torch, cs, fam, dim, dt, n):
    P, _ = synth.fill_host(fam, dim, synth.seed_for(41), n, dtype=dt)
    want, wfl = oracle.clip(P, n, *UNIT[dim], dim)
    dP = torch.from_numpy(P).cuda()
    g_out = Guarded(torch, 2 * dim, dP.shape[1], dP.dtype)
    g_fl = Guarded(torch, 0, n, torch.uint8)
    cs.clip(dP, n, *UNIT[dim], out=g_out.t, flags=g_fl.t)
    torch.cuda.synchronize()
    assert np.array_equal(g_fl.t.cpu().numpy(), wfl)
    assert np.array_equal(bits(g_out.t.cpu().numpy()[:, :n]), bits(want[:, :n]))
    assert g_out.untouched_from(n), "plane padding [n, ld) written"
    assert g_fl.untouched_from(n)


@pytest.mark.parametrize("dt,n,ndc", [(np.float32, 30011, True), (np.float64, 7001, False)])
def test_homog_guards(torch, cs, dt, n, ndc):
    P, _ = synth.fill_host(synth.HOMOG, 4, synth.seed_for(43), n, dtype=dt)
    dP = torch.from_numpy(P).cuda()
    rows = 6 if ndc else 8
    want, wfl = oracle.homog_clip(P, n, ndc=ndc)
    g_out = Guarded(torch, rows, dP.shape[1], dP.dtype)
    g_fl = Guarded(torch, 0, n, torch.uint8)
    cs.clip_homog(dP, n, ndc=ndc, out=g_out.t, flags=g_fl.t)
    torch.cuda.synchronize()
    assert np.array_equal(g_fl.t.cpu().numpy(), wfl)
    assert np.array_equal(bits(g_out.t.cpu().numpy()[:, :n]), bits(want[:rows, :n]))
    assert g_out.untouched_from(n) and g_fl.untouched_from(n)
    want, widx, wcnt, wfl = oracle.homog_compact(P, n, with_flags=True, ndc=ndc)
    b = compact_bufs(torch, cs, n, rows, dP.dtype)
    cs.clip_homog_compact(dP, n, ndc=ndc, bufs=b)
    torch.cuda.synchronize()
    c = int(b.count.item())
    assert c == wcnt
    assert np.array_equal(b.index.cpu().numpy()[:c], widx)
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :c]), bits(want[:rows, :c]))
    check_compact_guards(b, n, c)


def test_host_entry_guards(torch, cs):
    """The pipelined host-buffer entry (several chunks in flight): host outputs guarded."""
    n, dim = 50003, 2
    P, _ = synth.fill_host(synth.UNIFORM, dim, synth.seed_for(44), n)
    want, _, wcnt, wfl = oracle.compact(P, n, *UNIT[dim], dim, with_flags=True)
    h_in = torch.from_numpy(P).pin_memory()
    g_out = Guarded(torch, 2 * dim, P.shape[1], torch.float32, device="cpu", pin=True)
    g_fl = Guarded(torch, 0, n, torch.uint8, device="cpu", pin=True)
    c, _ = cs.clip_compact_host(h_in, n, *UNIT[dim], g_out.t, g_fl.t, chunk=8192)
    assert c == wcnt
    assert np.array_equal(g_fl.t.numpy(), wfl)
    assert np.array_equal(bits(g_out.t.numpy()[:, :c]), bits(want[:, :c]))
    assert g_out.untouched_from(c) and g_fl.untouched_from(n)
    assert np.array_equal(h_in.numpy(), P)


def test_tof_guards(torch, cs):
    from oracle import tof_oracle  # noqa: PLC0415
    ppf, nf = 777, 5
    d, I, r = synth.tof_host(synth.seed_for(45), nf, ppf=ppf)
    n = nf * ppf - 11                                   # last frame ragged
    d, I = d[:n].copy(), I[:n].copy()
    g_phi = Guarded(torch, 0, n, torch.float32)
    g_code = Guarded(torch, 0, n, torch.uint8)
    g_kept = Guarded(torch, 0, nf, torch.int32)
    cs.tof_range_phi(torch.from_numpy(d).cuda(), torch.from_numpy(I).cuda(), ppf,
                     torch.from_numpy(np.ascontiguousarray(r)).cuda(), phi=g_phi.t, code=g_code.t, kept=g_kept.t)
    torch.cuda.synchronize()
    wc, wp, wk = tof_oracle.tof_range_phi(d, I, ppf, r)
    assert np.array_equal(g_code.t.cpu().numpy(), wc)
    assert np.array_equal(g_kept.t.cpu().numpy(), wk)
    k = wc == 0
    assert np.abs(g_phi.t.cpu().numpy()[k].astype(np.float64) - wp[k]).max() <= 1e-6
    assert g_phi.untouched_from(n) and g_code.untouched_from(n) and g_kept.untouched_from(nf)


@pytest.mark.parametrize("F,H,W", [(2, 24, 32), (64, 12, 16)])   # grid-wide, then one block per frame
def test_cluster_guards(torch, cs, F, H, W):
    from oracle import cluster_oracle  # noqa: PLC0415
    from synth import scenes  # noqa: PLC0415
    z, ph, v, _ = scenes.batch(F, H, W, seed=77 + F)
    dz, dph, dv = (torch.from_numpy(a).cuda() for a in (z, ph, v.astype(np.uint8)))
    g_lab = Guarded(torch, 0, F * H * W, torch.int32)
    g_nreg = Guarded(torch, 0, F, torch.int32)
    g_rounds = Guarded(torch, 0, 1, torch.int32)
    need = int(cs.clip_cluster_workspace_bytes(F, H, W))
    g_ws = Guarded(torch, 0, need, torch.uint8)
    p = cs.TABLE1
    prm = cs.clip_merge_params(p["t_z"], p["t_phi"], p["alpha_z"], p["alpha_phi"])
    st = cs.clip_cluster_frames(dz.data_ptr(), dph.data_ptr(), dv.data_ptr(), F, H, W, ctypes.byref(prm), 1 << 30,
                                g_lab.t.data_ptr(), g_nreg.t.data_ptr(), g_rounds.t.data_ptr(), g_ws.t.data_ptr(),
                                need, None)
    assert st == cs.CLIP_OK
    torch.cuda.synchronize()
    L = g_lab.t.view(F, H, W).cpu().numpy()
    for f in (0, F - 1):
        wl, wr, _, _ = cluster_oracle.cluster(z[f], ph[f], v[f])
        assert np.array_equal(L[f], wl)
        assert int(g_nreg.t[f]) == len(wr)
    assert g_lab.untouched_from(F * H * W) and g_nreg.untouched_from(F) and g_rounds.untouched_from(1)
    assert g_ws.untouched_from(need), "cluster workspace overrun"
