"""One warm-up call and one measured call of every per-config report record
(tests/test_report_gpu.py RECORDS), in that order, for an ncu launch list: prints one JSON line
per record with its launch count, so tools/ncu_bytes.py can cut the list into calls."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1505_00996_b200 as fgf  # noqa: E402
import synth  # noqa: E402
from test_report_gpu import RECORDS  # noqa: E402

torch.cuda.set_device(0)
out = []
for cfg, s_over, _ in RECORDS:
    c = synth.CONFIGS[cfg]
    prm = synth.params(cfg, **({} if s_over is None else {"s": s_over}))
    B = 32 if (cfg == 4 and prm["s"] == 1) else c["batch"]
    I, p = synth.make_batch(cfg, "cuda", batch=B)
    q = torch.empty((B, c["C_p"], c["H"], c["W"]), device="cuda")
    nb = fgf.fgf_workspace_bytes(B, c["H"], c["W"], c["C_I"], c["C_p"], prm["r"], prm["s"])
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):   # warm-up call, measured call (both in the launch list)
        fgf.fgf_filter_ws(I, p, q, B, c["H"], c["W"], c["C_I"], c["C_p"], prm["r"], prm["eps"],
                          prm["s"], prm["sub_mode"], ws, nb, torch.cuda.current_stream())
        torch.cuda.synchronize()
    out.append({"key": f"{c['name']}_s{prm['s']}", "launches": fgf.fgf_last_launch_count()})
    del I, p, q, ws
    torch.cuda.empty_cache()
print(json.dumps(out))
