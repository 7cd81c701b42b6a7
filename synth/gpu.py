"""GPU twin of the synthetic generator (ctypes over synth/libsynth.so). Input generation only."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import torch

from . import (KIND_NORM, MASK_E, MASK_R, S_EXP, S_MASK, S_PERT, S_ROW, S_VAL, EXPERT_F, ROW_Q, Manifest, h, key,
               threshold, bf16_table, table, ONE, DTYPE_BF16, DTYPE_FP8)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cu")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", _SRC, "-o", _LIB])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = ctypes.CDLL(_LIB)
        P, u64, i32, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32
        L.synth_fill_old.argtypes = [P, u64, i32, u64, P, P]
        L.synth_fill_new.argtypes = [P, P, u64, i32, i32, u64, u64, u64, u64, u64, u64, P]
        L.synth_toggle.argtypes = [P, P, P, P, u32, P, P]
        L.synth_fill_old8.argtypes = [P, u64, i32, u64, P, P]
        L.synth_fill_new8.argtypes = [P, P, u64, i32, i32, u64, u64, u64, u64, u64, u64, P]
        L.synth_fill_new_jobs.argtypes = [P, P, P, u64, u64, P]
        L.synth_fill_new_jobs.restype = ctypes.c_int
        for f in (L.synth_fill_old, L.synth_fill_new, L.synth_toggle, L.synth_fill_old8, L.synth_fill_new8):
            f.restype = i32
        _lib = L
    return _lib


_tables = {}


def _table(device, dtype: int = DTYPE_BF16) -> torch.Tensor:
    k = (str(device), dtype)
    if k not in _tables:
        tb = table(dtype)
        _tables[k] = torch.from_numpy(tb.copy() if tb.dtype == np.uint8 else tb.view(np.int16).copy()).to(device)
    return _tables[k]


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def arena(manifest: Manifest, device, dtype=torch.int16):
    """One flat tensor + per-tensor views (every numel is a multiple of 8 -> 16 B aligned views)."""
    total = manifest.total
    buf = torch.empty(max(total, 1), dtype=dtype, device=device)
    views, off = [], 0
    for t in manifest.tensors:
        views.append(buf[off:off + t.numel])
        off += t.numel
    return buf, views


def fill_old(views, manifest: Manifest, seed: int, tid0: int = 0, dtype: int = DTYPE_BF16):
    tab = _table(views[0].device, dtype) if views else None
    for k, (v, t) in enumerate(zip(views, manifest.tensors)):
        f = lib().synth_fill_old8 if dtype == DTYPE_FP8 else lib().synth_fill_old
        rc = f(ctypes.c_void_p(v.data_ptr()), v.numel(), ONE[dtype] if t.kind == KIND_NORM else 0,
                                  key(S_VAL, seed, tid0 + k), ctypes.c_void_p(tab.data_ptr()), _s())
        assert rc == 0


def fill_new(old_views, new_views, manifest: Manifest, seed: int, rho: float, mask: int = 0, tid0: int = 0):
    for k, (o, n, t) in enumerate(zip(old_views, new_views, manifest.tensors)):
        tid = tid0 + k
        mode, active, thr = 0, 1, threshold(rho)
        key_row, thr_row, cols = 0, 0, 1
        if mask == MASK_R and len(t.shape) == 2:
            mode, thr = 1, threshold(min(1.0, rho / ROW_Q))
            key_row, thr_row, cols = key(S_ROW, seed, tid), threshold(ROW_Q), t.cols
        elif mask == MASK_E and t.expert >= 0:
            e = np.array([t.expert], np.uint64)
            active = int((h(S_EXP, seed, t.layer, e) >> np.uint64(32))[0] < np.uint64(threshold(EXPERT_F)))
            thr = threshold(min(1.0, rho / EXPERT_F))
        f = lib().synth_fill_new8 if o.element_size() == 1 else lib().synth_fill_new
        rc = f(ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(n.data_ptr()), o.numel(), mode,
                                  active, key(S_MASK, seed, tid), thr, key(S_PERT, seed, tid), key_row, thr_row,
                                  cols, _s())
        assert rc == 0


class FillNewPlan:
    """fill_new over many tensors in ONE launch (bench streaming mode): the per-tensor parameters of
    fill_new in a device job table, tiles of 1 Mi elements; bit-identical to calling fill_new per tensor."""
    TILE = 1 << 20

    def __init__(self, old_views, new_views, manifest: Manifest, seed: int, rho: float, mask: int = 0,
                 tid0: int = 0):
        assert all(o.element_size() == 2 for o in old_views)
        jobs, tj, to = [], [], []
        for k, (o, n, t) in enumerate(zip(old_views, new_views, manifest.tensors)):
            tid = tid0 + k
            mode, active, thr = 0, 1, threshold(rho)
            key_row, thr_row, cols = 0, 0, 1
            if mask == MASK_R and len(t.shape) == 2:
                mode, thr = 1, threshold(min(1.0, rho / ROW_Q))
                key_row, thr_row, cols = key(S_ROW, seed, tid), threshold(ROW_Q), t.cols
            elif mask == MASK_E and t.expert >= 0:
                e = np.array([t.expert], np.uint64)
                active = int((h(S_EXP, seed, t.layer, e) >> np.uint64(32))[0] < np.uint64(threshold(EXPERT_F)))
                thr = threshold(min(1.0, rho / EXPERT_F))
            # FillJob: 2 pointers, 7 u64, 2 int32 (80 bytes)
            jobs.append([o.data_ptr(), n.data_ptr(), o.numel(), key(S_MASK, seed, tid), thr, key(S_PERT, seed, tid),
                         key_row, thr_row, cols, (active << 32) | mode])
            for e0 in range(0, o.numel(), self.TILE):
                tj.append(len(jobs) - 1)
                to.append(e0)
        dev = old_views[0].device
        a = np.array(jobs, dtype=np.uint64).reshape(-1, 10) if jobs else np.zeros((0, 10), np.uint64)
        self.jobs = torch.from_numpy(a.view(np.int64).copy()).to(dev)
        self.tile_job = torch.tensor(tj or [0], dtype=torch.int32, device=dev)
        self.tile_off = torch.tensor(to or [0], dtype=torch.int64, device=dev)
        self.n_tiles = len(tj)

    def run(self):
        rc = lib().synth_fill_new_jobs(ctypes.c_void_p(self.jobs.data_ptr()), ctypes.c_void_p(self.tile_job.data_ptr()),
                                       ctypes.c_void_p(self.tile_off.data_ptr()), self.n_tiles, self.TILE, _s())
        assert rc == 0


def toggle(y_ptrs: torch.Tensor, I: torch.Tensor, V: torch.Tensor, counts: torch.Tensor, T: int, scratch: torch.Tensor):
    """Bench 'optimizer step': Y[t][I] = V ^ 1 (V = Y[I] at extraction) for the positions of the last sync
    (scratch: >= T+1 int64)."""
    rc = lib().synth_toggle(ctypes.c_void_p(y_ptrs.data_ptr()), ctypes.c_void_p(I.data_ptr()),
                            ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(counts.data_ptr()), T,
                            ctypes.c_void_p(scratch.data_ptr()), _s())
    assert rc == 0
