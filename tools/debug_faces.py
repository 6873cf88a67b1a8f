"""Print the golden faces where the FAST variant departs from the reference."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1307_0491_b200 import abi, native
data = np.load(os.path.join(ROOT, "tests/golden/golden.npz"))
meta = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))
np.set_printoptions(precision=17, linewidth=200)
for case in ["faces_ag0p3", "faces_ag0p001", "faces_ag0", "faces_ag5"]:
    for axis in (0, 1):
        p = abi.make_problem(2, 4, 4, 1.0, 1.0, a_g=meta["cases"][case]["a_g"])
        L, R = data[f"{case}_ax{axis}_L"], data[f"{case}_ax{axis}_R"]
        ref, info = data[f"{case}_ax{axis}_out"], data[f"{case}_ax{axis}_info"]
        out = native.faces(p, L, R, axis, abi.VARIANT_FAST)
        err = np.max(np.abs(out - ref) / np.maximum(1, np.abs(ref)), axis=1)
        bad = np.nonzero(err > 1e-11)[0]
        print(case, axis, "bad", len(bad), "of", len(err), "max", err.max())
        for k in bad[:6]:
            print("  k", k, "err", err[k], "info(a,b,enl,branch)", info[k])
            print("    L", L[k], "R", R[k])
            print("    ref", ref[k]); print("    got", out[k])
