"""Write tests/golden/tiny_seed.json by calling only `oracle/` and `synth/`.

Seed acceptance: the first seed >= 0 whose oracle
(fp64) greedy run has min over steps of (top1 - top2) >= 0.1, so bf16 rounding
on the GPU path cannot flip a token.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import TINY, gen_weights, tiny_request  # noqa: E402
from oracle.vlm import OracleWeights, generate  # noqa: E402


def main():
    for seed in range(0, 100):
        bits = gen_weights(TINY, seed)
        req = tiny_request(TINY, seed)
        out = generate(OracleWeights(bits, np.float64), req.pixels, req.prompt_ids, req.gen_len, TINY)
        m = float(out["margins"].min())
        print(seed, m)
        if m >= 0.1:
            rec = {"seed": seed, "min_margin": m, "tokens": out["tokens"].tolist(),
                   "rule": "first seed >= 0 with min top-2 margin >= 0.1 (SURVEY.md 8(c) c5 row 8)",
                   "written_by": "scripts/make_golden.py (oracle/ + synth/ only)"}
            with open(os.path.join(ROOT, "tests", "golden", "tiny_seed.json"), "w") as f:
                json.dump(rec, f, indent=1)
            return


if __name__ == "__main__":
    main()
