"""The multi-rank C band path (fgf_filter_band_ex) executed by several PROCESSES on one GPU:
each rank is its own process with its own band rows, workspace, stream and communicator, and
the halos travel through libfgf.so's own NCCL call sequence (ncclGroupStart / ncclSend /
ncclRecv / ncclGroupEnd per plane, rank +- 1), served by tests/nccl_shim.cpp in place of
NCCL (one GPU here: NCCL itself refuses two ranks on one device).  The assembled bands must
equal the one-process loopback of the same plan bit for bit, the whole-image filter to
fp32 rounding and the oracle to the BASELINE tolerance."""
from __future__ import annotations

import ctypes
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import paper_1505_00996_b200 as fgf
from paper_1505_00996_b200 import bands

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SHIM = os.path.join(HERE, "libnccl_shim.so")


def _unique_id() -> bytes:
    uid = ctypes.create_string_buffer(128)
    assert ctypes.CDLL(SHIM).ncclGetUniqueId(uid) == 0
    return uid.raw


def _run_ranks(nranks, C_I, C_p, H, W, r, eps, s, sub, mode, seed, self_g, tmp_path):
    raw = _unique_id()
    uid, rdv = raw.hex(), raw.rstrip(b"\0").decode()
    env = dict(os.environ, FGF_DEV="1", FGF_NCCL_LIB=SHIM)
    procs, outs = [], []
    for k in range(nranks):
        out = str(tmp_path / f"q{k}.npy")
        outs.append(out)
        args = [uid, k, nranks, C_I, C_p, H, W, r, eps, s, sub, mode, seed, int(self_g), out]
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "band_rank_worker.py")]
                                      + [str(x) for x in args], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for pr in procs:
        try:
            o, _ = pr.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for x in procs:
                x.kill()
            raise
        logs.append((pr.returncode, o.decode(errors="replace")[-2000:]))
    for k, (rc, log) in enumerate(logs):
        assert rc == 0, f"rank {k} failed:\n{log}"
    # the halos really travelled between the processes: one message per send, two calls,
    # planes x (up + down) per interior rank
    msgs = [m for m in os.listdir(rdv) if m.startswith("m_") and not m.endswith(".tmp")]
    shutil.rmtree(rdv, ignore_errors=True)
    assert len(msgs) >= 2 * 2 * (nranks - 1), msgs
    return np.concatenate([np.load(o) for o in outs], axis=1)[None]   # [1, C_p, H, W]


@pytest.mark.parametrize("mode", [fgf.FGF_BAND_SINGLE, fgf.FGF_BAND_TWO_STEP])
@pytest.mark.parametrize("nranks,C_I,C_p,s,sub,self_g,H,W", [(2, 1, 1, 4, 0, False, 1200, 1032),
                                                            (4, 1, 1, 4, 0, True, 1200, 1032),
                                                            (3, 3, 1, 2, 1, False, 1200, 1032),
                                                            (3, 3, 3, 4, 0, False, 1200, 1032),
                                                            (8, 1, 1, 4, 0, False, 4096, 1536),
                                                            (5, 1, 2, 1, 0, False, 1001, 517)])
def test_band_processes_match_loopback_and_oracle(nranks, C_I, C_p, s, sub, self_g, H, W, mode,
                                                  tmp_path):
    """(8 ranks, r = 32, s = 4: config 4b's split and window on a 4096-row image; 5 ranks at
    s = 1 with ragged bands and two p channels)"""
    if not os.path.exists(SHIM):
        pytest.fail("tests/libnccl_shim.so missing: run make")
    r, eps, seed = 32, 0.01, 41 + nranks
    q = _run_ranks(nranks, C_I, C_p, H, W, r, eps, s, sub, mode, seed, self_g, tmp_path)
    g = torch.Generator(device="cuda").manual_seed(seed)
    I = torch.rand((1, C_I, H, W), device="cuda", generator=g)
    p = I if self_g else torch.rand((1, C_p, H, W), device="cuda", generator=g)
    qt = torch.from_numpy(q).cuda()
    # the same plan in one process (halos copied between the bands' buffers)
    nb = fgf.fgf_bands_loopback_workspace_bytes(H, W, C_I, C_p, r, s, nranks)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    q_loop = torch.empty((1, C_p, H, W), device="cuda")
    fgf.fgf_filter_bands_loopback(I, p, q_loop, H, W, C_I, C_p, r, eps, s, sub, nranks, ws, nb,
                                  torch.cuda.current_stream(), mode=mode)
    q_whole = fgf.filter(I, p, r, eps, s, sub)
    torch.cuda.synchronize()
    assert torch.equal(qt, q_loop)
    assert float((qt - q_whole).abs().max()) < 1e-5
    ref = oracle.fast_guided_filter(I.cpu().numpy(), p.cpu().numpy(), r, eps, s, sub)
    assert float(np.abs(q.astype(np.float64) - ref).max()) < 1e-4
    assert bands.plan_band(H, W, r, s, nranks, nranks - 1).Y1 == H
