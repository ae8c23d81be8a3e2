"""One rank of the multi-process band test (tests/test_band_multirank_gpu.py): builds the
seeded full image, keeps its own band rows, runs fgf_filter_band_ex through the communicator
of the NCCL stand-in (FGF_DEV=1, FGF_NCCL_LIB=tests/libnccl_shim.so) and saves q of its rows.
usage: python band_rank_worker.py <uid_hex> <rank> <nranks> <C_I> <C_p> <H> <W> <r> <eps> <s>
       <sub> <mode> <seed> <self_guided> <out.npy>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00996_b200 as fgf  # noqa: E402
from paper_1505_00996_b200 import bands  # noqa: E402


def main(a):
    uid = bytes.fromhex(a[0])
    rank, nranks, C_I, C_p, H, W, r = (int(x) for x in a[1:8])
    eps = float(a[8])
    s, sub, mode, seed, self_g = (int(x) for x in a[9:14])
    out = a[14]
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(seed)
    I = torch.rand((1, C_I, H, W), device="cuda", generator=g)
    p = I if self_g else torch.rand((1, C_p, H, W), device="cuda", generator=g)
    pl = bands.plan_band(H, W, r, s, nranks, rank)
    rows = pl.Y1 - pl.Y0
    I_own = I[0, :, pl.Y0:pl.Y1].contiguous()
    p_own = I_own if self_g else p[0, :, pl.Y0:pl.Y1].contiguous()
    q_own = torch.empty((C_p, rows, W), device="cuda")
    comm = fgf.fgf_nccl_comm_init(uid, rank, nranks)
    nb = fgf.fgf_band_workspace_bytes(H, W, pl.Y0, rows, C_I, C_p, r, s, nranks)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(2):   # twice: the second call reuses the library's band streams
            fgf.fgf_filter_band_ex(I_own, p_own, q_own, H, W, pl.Y0, rows, C_I, C_p, r, eps, s,
                                   sub, mode, comm, rank, nranks, ws, nb, st)
    st.synchronize()
    assert fgf.fgf_nccl_check(comm) == fgf.FGF_OK
    fgf.fgf_nccl_comm_destroy(comm)
    np.save(out, q_own.cpu().numpy())


if __name__ == "__main__":
    main(sys.argv[1:])
