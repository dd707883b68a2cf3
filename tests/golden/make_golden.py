"""Write tests/golden/cfg1_oracle.json.  Calls ONLY oracle/ (and the seeded
input generator); never the CUDA path.  Run: python tests/golden/make_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from bie_inputs import make_config  # noqa: E402

d = make_config(1)
u = oracle.apply(d["centres"], d["radii"], 4, 1.0, d["f"], d["q"])
with open(os.path.join(HERE, "cfg1_oracle.json"), "w") as fh:
    json.dump({"source": "oracle.apply on BASELINE.json configs[0] (seed 0), p=4, mu=1",
               "u": [[float(v) for v in row] for row in u]}, fh, indent=0)
print("wrote", os.path.join(HERE, "cfg1_oracle.json"))
