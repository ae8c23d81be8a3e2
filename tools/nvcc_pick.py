"""Compile one CUDA translation unit several times and keep the object whose code for a given
kernel uses the uniform datapath most.

nvcc's --split-compile NVVM output is not deterministic (the same source gives different PTX
from run to run), and for the default K13 variant the two outcomes differ in speed: with its
loop and ring indices on the uniform datapath (~540 uniform SASS instructions) K13 takes
3.91 ms on config 4, otherwise (~200, or ~60 unsplit) 4.1-4.2 ms (build).  This
picks the former: up to --tries compiles, --par at a time, keeping the one with the most
uniform instructions and stopping after the first round that reaches --want (the two outcomes
of the current source: ~515 uniform instructions / 127 registers, fast, and ~426 / 102).

usage: python tools/nvcc_pick.py --out build/x.o --kernel <mangled name> [--tries 8]
                                 [--want 500] [--par 4] -- nvcc <args without -o>
"""
import argparse
import os
import re
import shutil
import subprocess
import sys
import tempfile


def uniform_count(obj, kernel):
    if shutil.which("cuobjdump") is None:   # no disassembler: take the compile as it comes
        return 1 << 30
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    n, on, found = 0, False, False
    for line in out.splitlines():
        if "Function :" in line:
            on = line.strip().endswith(kernel)
            found = found or on
            continue
        if on:
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?(\S+)", line)
            if m and m.group(2).startswith("U"):
                n += 1
    if not found:
        sys.exit(f"nvcc_pick: kernel {kernel} not in {obj} (Makefile K13_V3 out of date?)")
    return n


def main():
    argv = sys.argv[1:]
    if "--" not in argv:
        sys.exit(__doc__)
    k = argv.index("--")
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--tries", type=int, default=8)
    ap.add_argument("--want", type=int, default=500)
    ap.add_argument("--par", type=int, default=4)
    a = ap.parse_args(argv[:k])
    cmd = argv[k + 1:]
    env = {x: y for x, y in os.environ.items() if x not in ("MAKEFLAGS", "MFLAGS")}
    best, best_n = None, -1
    tmp = tempfile.mkdtemp(prefix="nvcc_pick_")
    try:
        # compiles run a.par at a time (each is one single-threaded nvcc); stop after the first
        # round that reaches --want
        t = 0
        while t < a.tries:
            procs = []
            for _ in range(min(a.par, a.tries - t)):
                obj = os.path.join(tmp, f"try{t}.o")
                procs.append((t, obj, subprocess.Popen(cmd + ["-o", obj], env=env)))
                t += 1
            codes = [(k, obj, pr.wait()) for k, obj, pr in procs]   # all finished first
            for k, obj, rc in codes:
                if rc != 0:
                    sys.exit(f"nvcc_pick: compile {k} failed")
                n = uniform_count(obj, a.kernel)
                print(f"nvcc_pick: try {k}: {n} uniform instructions in {a.kernel[:48]}...", file=sys.stderr)
                if n > best_n:
                    best, best_n = obj, n
            if best_n >= a.want:
                break
        shutil.copyfile(best, a.out)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
