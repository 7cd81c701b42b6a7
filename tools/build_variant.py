"""Build an A/B variant of libsparsesync.so with extra nvcc defines (dev tool; load it with SS_LIB=<path>).
usage: python tools/build_variant.py <tag> [--git REV] -DNAME=VALUE [...]
       -> paper_2605_07330_b200/build/libsparsesync_<tag>.so
--git REV builds the csrc/ of that revision (checked out next to csrc/, so its relative includes resolve)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_07330_b200 import build as b  # noqa: E402


def main():
    tag, defs = sys.argv[1], sys.argv[2:]
    srcs = b._sources()
    if "--git" in defs:
        rev = defs[defs.index("--git") + 1]
        defs = [d for d in defs if d not in ("--git", rev)]
        cdir = os.path.join(os.path.dirname(b.CSRC), "csrc_" + tag)
        os.makedirs(cdir, exist_ok=True)
        names = subprocess.check_output(["git", "ls-tree", "--name-only", f"{rev}:paper_2605_07330_b200/csrc"],
                                        cwd=ROOT, text=True).split()
        for n in names:
            with open(os.path.join(cdir, n), "w") as f:
                f.write(subprocess.check_output(["git", "show", f"{rev}:paper_2605_07330_b200/csrc/{n}"], cwd=ROOT,
                                                text=True))
        srcs = sorted(os.path.join(cdir, n) for n in names if n.endswith(".cu"))
    out_dir = os.path.join(b.BUILD, "var_" + tag)
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in srcs:
        o = os.path.join(out_dir, os.path.basename(src)[:-3] + ".o")
        subprocess.check_call([b.NVCC, *b.FLAGS, *defs, "-c", src, "-o", o])
        objs.append(o)
    lib = os.path.join(b.BUILD, f"libsparsesync_{tag}.so")
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
