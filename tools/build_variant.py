"""Build an A/B variant of libsparsesync.so with extra nvcc defines (dev tool; load it with SS_LIB=<path>).
usage: python tools/build_variant.py <tag> -DNAME=VALUE [...]  ->  paper_2605_07330_b200/build/libsparsesync_<tag>.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_07330_b200 import build as b  # noqa: E402


def main():
    tag, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(b.BUILD, "var_" + tag)
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in b._sources():
        o = os.path.join(out_dir, os.path.basename(src)[:-3] + ".o")
        subprocess.check_call([b.NVCC, *b.FLAGS, *defs, "-c", src, "-o", o])
        objs.append(o)
    lib = os.path.join(b.BUILD, f"libsparsesync_{tag}.so")
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
