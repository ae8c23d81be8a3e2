"""Save q of a few workloads with the library FGF_LIB_NAME selects (A/B bit-identity checks
of two builds): python tools/bitcmp.py out.pt; python tools/bitcmp.py --cmp a.pt b.pt"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "--cmp":
    a, b = torch.load(sys.argv[2]), torch.load(sys.argv[3])
    for k in a:
        print(k, "bit-identical" if torch.equal(a[k], b[k]) else
              f"DIFFERENT max {float((a[k] - b[k]).abs().max()):.3e}")
    sys.exit(0)

import paper_1505_00996_b200 as fgf  # noqa: E402
import synth  # noqa: E402

out = {}
for cfg, kw in [(1, {}), (2, {}), (3, {"batch": 2}), (0, {}), (5, {"batch": 1, "H": 4096, "W": 4096}) if False else (4, {"batch": 2})]:
    I, p = synth.make_batch(cfg, "cuda", **kw)
    prm = synth.params(cfg)
    out[f"cfg{cfg}"] = fgf.filter(I, p, **prm).cpu()
    if cfg == 1:
        out["cfg1_s1"] = fgf.filter(I, p, **dict(prm, s=1)).cpu()
        out["cfg1_block"] = fgf.filter(I, p, **dict(prm, sub_mode=1)).cpu()
torch.save(out, sys.argv[1])
print("saved", list(out))
