"""Oracle O14 flagged-pixel fractions per configuration (reading Q20 bands, CPU only).
usage: python tools/flag_stats.py [out.json]"""
import json
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

CASES = [("C1", 1.0, [0]), ("C2", 1.0, [0]), ("C3", 0.1, [0, 1, 2, 3, 4]), ("C4", 0.05, [0, 1, 2]),
         ("C5", 0.02, [0, 9])]


def main():
    out = []
    for cfg, scale, views in CASES:
        sc, vs = synth.make_config(cfg, scale=scale)
        for i in views:
            t = time.time()
            o = oracle.render(sc, vs[i], a_min=0.5, binning="tight")
            fl = o["flags"]
            n = fl.size
            r = dict(config=cfg, scale=scale, view=i, width=vs[i].width, height=vs[i].height,
                     evals_per_px=o["evals"] / n, blends_per_px=o["blends"] / n,
                     flagged_frac=float((fl != 0).sum()) / n, alpha_band=float((fl & 1).astype(bool).sum()) / n,
                     t_band=float((fl & 2).astype(bool).sum()) / n, amin_band=float((fl & 4).astype(bool).sum()) / n,
                     oracle_s=round(time.time() - t, 1))
            print(json.dumps(r), flush=True)
            out.append(r)
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
