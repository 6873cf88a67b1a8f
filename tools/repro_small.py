"""Small FAST run for sanitizers: rand48x32 golden case, 60 steps."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1307_0491_b200 import abi, native
from conftest import problem_from_meta, normwise
data = np.load(os.path.join(ROOT, "tests/golden/golden.npz"))
meta = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))
m = meta["cases"]["rand48x32"]
p = problem_from_meta(m)
try:
    out, t, n, log = native.run(p, data["rand48x32_init"], max_steps=m["max_steps"], variant=abi.VARIANT_FAST)
    print("steps", n, "err", normwise(out, data["rand48x32_final"]))
except Exception as e:
    print("raised", type(e).__name__, e)
