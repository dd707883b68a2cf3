#!/usr/bin/env python
"""Compile only the far-field kernel instantiations (no libbie build) and run
the register-file read model (tools/sass_rf_model.py) on each hot inner loop.
A quick CPU-side check of an edit to k_nbody.cuh before spending GPU time
(the model tracked a measured 0.9 % apply slowdown to 0.1 %).
Usage: python tools/nbody_rf.py [-D...]"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INST = {
    "apply": "k_nbody<8, 64, 64, 3, false, 1, 2>",
    "off": "k_nbody<7, 64, 64, 3, true, 1, 2>",
    "K": "k_nbody<7, 64, 64, 3, false, 1, 2, 1>",
    "apply_const": "k_nbody_c<8, 64, 4, 0, false>",   # sources as constant-bank operands
    "off_const": "k_nbody_c<8, 64, 2, 0, true>",
}


def main():
    extra = sys.argv[1:]
    if os.environ.get("NBODY_INST"):  # e.g. "k_nbody<4, 64, 64, 3, false, 1, 4>;k_nbody<...>"
        INST.clear()
        INST.update({str(i): v for i, v in enumerate(os.environ["NBODY_INST"].split(";"))})
    src = '#include "k_nbody.cuh"\n#include "k_nbody_c.cuh"\nnamespace bie {\n' + "".join(
        f"template __global__ void {v}(const {'NbodyCArgs' if v.startswith('k_nbody_c') else 'NbodyArgs'});\n"
        for v in INST.values()) + "}\n"
    with tempfile.TemporaryDirectory() as td:
        cu = os.path.join(td, "k.cu")
        open(cu, "w").write(src)
        cub = os.path.join(td, "k.cubin")
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin",
                            "-Xptxas", "-v", "-I", os.environ.get("NBODY_SRC", os.path.join(ROOT, "paper_1707_06551_b200", "csrc")), *extra,
                            "-o", cub, cu], capture_output=True, text=True)
        if r.returncode:
            print(r.stderr)
            sys.exit(1)
        regs = re.findall(r"Compiling entry function '(\S+)'.*?Used (\d+) registers", r.stderr, re.S)
        sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
        for f in sass.split("Function : ")[1:]:
            name = f.split("\n")[0].strip()
            pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
            ins = [(int(m.group(1), 16), m.group(2)) for l in f.split("\n") for m in [pat.search(l)] if m]
            fs = os.path.join(td, "f.sass")
            open(fs, "w").write(f)
            reg = dict(regs).get(name, "?")
            for a, s in ins:
                m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", s)
                if not m:
                    continue
                lo = int(m.group(1), 16)
                body = [x for aa, x in ins if lo <= aa <= a]
                nfp = sum(1 for x in body if re.match(r"(@\S+\s+)?D(FMA|MUL|ADD)", x))
                if lo < a and nfp >= int(os.environ.get("NBODY_MINFP", "400")) and len(body) < 1400:
                    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_rf_model.py"), fs,
                                          hex(lo), hex(a)], capture_output=True, text=True).stdout.split("\n")[0]
                    print(f"{name[:60]:60s} regs {reg} loop {len(body)} instr: {out}")


if __name__ == "__main__":
    main()
