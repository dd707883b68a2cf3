#!/usr/bin/env python
"""Run tools/sass_rf_model.py on every long inner loop of every k_nbody
instantiation in a binary: python tools/rf_report.py <binary>"""
import re
import subprocess
import sys

txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in txt.split("Function : ")[1:]:
    name = f.split("\n")[0].strip()
    if "k_nbody" not in name:
        continue
    pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
    ins = [(int(m.group(1), 16), m.group(2)) for l in f.split("\n") for m in [pat.search(l)] if m]
    with open("/tmp/_f.sass", "w") as fh:
        fh.write(f)
    for a, s in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", s)
        if m and int(m.group(1), 16) < a and a - int(m.group(1), 16) > 0x800:
            lo = int(m.group(1), 16)
            out = subprocess.run([sys.executable, "tools/sass_rf_model.py", "/tmp/_f.sass", hex(lo), hex(a)],
                                 capture_output=True, text=True).stdout.split("\n")[0]
            print(name[:64], hex(lo), hex(a), out)
