"""Test-only native helpers (built on demand; never imported by the product)."""
import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SPIN_SO = os.path.join(HERE, "libspin.so")


def build_spin() -> str:
    src = os.path.join(HERE, "spin.cu")
    if not os.path.exists(SPIN_SO) or os.path.getmtime(SPIN_SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SPIN_SO, src])
    return SPIN_SO


def spin_lib():
    L = ctypes.CDLL(build_spin())
    L.spin_start.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.spin_start.restype = ctypes.c_int
    L.spin_started.argtypes = []
    L.spin_started.restype = ctypes.c_int
    L.spin_release.argtypes = []
    L.spin_release.restype = None
    return L
