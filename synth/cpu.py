"""CPU twin of the synthetic generator (ctypes over synth/libsynth_cpu.so). Input generation only."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import (KIND_NORM, MASK_E, MASK_R, S_EXP, S_MASK, S_PERT, S_ROW, S_VAL, EXPERT_F, ROW_Q, Manifest, h, key,
               threshold, bf16_table, table, ONE, DTYPE_BF16, DTYPE_FP8)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen_cpu.c")
_LIB = os.path.join(_HERE, "libsynth_cpu.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", _SRC, "-o", _LIB])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        L.synth_cpu_fill_old.argtypes = [P, u64, i32, u64, P]
        L.synth_cpu_fill_new.argtypes = [P, P, u64, i32, i32, u64, u64, u64, u64, u64, u64]
        L.synth_cpu_fill_old.restype = None
        L.synth_cpu_fill_new.restype = None
        L.synth_cpu_fill_old8.argtypes = [P, u64, i32, u64, P]
        L.synth_cpu_fill_new8.argtypes = [P, P, u64, i32, i32, u64, u64, u64, u64, u64, u64]
        L.synth_cpu_fill_old8.restype = None
        L.synth_cpu_fill_new8.restype = None
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def generate(manifest: Manifest, seed: int = 0, rho: float = 0.01, mask: int = 0, tid0: int = 0,
             dtype: int = DTYPE_BF16):
    """Same output as synth.generate (numpy), ~50x faster."""
    tab = table(dtype)
    olds, news = [], []
    for k, t in enumerate(manifest.tensors):
        tid = tid0 + k
        e8 = dtype == DTYPE_FP8
        o = np.empty(t.numel, np.uint8 if e8 else np.uint16)
        n = np.empty(t.numel, np.uint8 if e8 else np.uint16)
        if t.numel:
            (lib().synth_cpu_fill_old8 if e8 else lib().synth_cpu_fill_old)(_p(o), t.numel, ONE[dtype] if t.kind == KIND_NORM else 0,
                                     key(S_VAL, seed, tid), _p(tab))
            mode, active, thr = 0, 1, threshold(rho)
            key_row, thr_row, cols = 0, 0, 1
            if mask == MASK_R and len(t.shape) == 2:
                mode, thr = 1, threshold(min(1.0, rho / ROW_Q))
                key_row, thr_row, cols = key(S_ROW, seed, tid), threshold(ROW_Q), t.cols
            elif mask == MASK_E and t.expert >= 0:
                e = np.array([t.expert], np.uint64)
                active = int((h(S_EXP, seed, t.layer, e) >> np.uint64(32))[0] < np.uint64(threshold(EXPERT_F)))
                thr = threshold(min(1.0, rho / EXPERT_F))
            (lib().synth_cpu_fill_new8 if e8 else lib().synth_cpu_fill_new)(
                _p(o), _p(n), t.numel, mode, active, key(S_MASK, seed, tid), thr,
                                     key(S_PERT, seed, tid), key_row, thr_row, cols)
        olds.append(o)
        news.append(n)
    return olds, news
