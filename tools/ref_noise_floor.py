"""The reference's own rounding sensitivity on a config: compare two reference
runs saved by tools/ref_solve_save.py, one from the stock build (oracle/_ref)
and one from a rounding-variant build of the same sources
(make -C oracle OUT=_ref/fma EXTRA="-mavx2 -mfma -ffp-contract=fast", selected
with OPTCON_REF_LIB). The differences are the floor any other correct
implementation can be expected to reach on that config.

    python tools/ref_noise_floor.py stock.npz variant.npz [--out report.json]
"""
import argparse
import json

import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("stock")
ap.add_argument("variant")
ap.add_argument("--label", default="")
ap.add_argument("--out", default=None)
a = ap.parse_args()
s, v = np.load(a.stock), np.load(a.variant)


def rel(k):
    return float(np.linalg.norm(s[k] - v[k]) / max(np.linalg.norm(s[k]), 1e-300))


rep = dict(label=a.label, level=int(s["level"]),
           rel_u=rel("u"), rel_y=rel("y"),
           rel_J=float(abs(s["objective"] - v["objective"]) / abs(s["objective"])),
           nli=[int(s["nli"]), int(v["nli"])],
           lin_stock=[int(x) for x in s["lin"]], lin_variant=[int(x) for x in v["lin"]],
           seconds=[float(s["seconds"]), float(v["seconds"])])
print(json.dumps(rep))
if a.out:
    try:
        with open(a.out) as f:
            allr = json.load(f)
    except (OSError, ValueError):
        allr = []
    allr = [r for r in allr if not (r["label"] == rep["label"] and r["level"] == rep["level"])]
    allr.append(rep)
    with open(a.out, "w") as f:
        json.dump(allr, f, indent=1)
