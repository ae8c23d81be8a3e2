"""CPU test double of the band-path compute stages, built only from the pinned oracle and the
brute-force interpolation matrices, so the band HOST logic (plan, halo exchange, assembly,
global offsets) can be tested with gloo on CPU against the whole-image oracle."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from tests import brute


class OracleBackend:
    def subsample(self, x, s, sub_mode):
        xn = x.double().numpy()
        B, C = xn.shape[:2]
        out = np.stack([np.stack([oracle.subsample(xn[b, c], s, sub_mode) for c in range(C)])
                        for b in range(B)])
        return torch.from_numpy(out)

    def lowres_mean(self, Is, ps, R, eps):
        # steps 2-5 on the given planes = the oracle's stages 1-5 at s = 1 with radius R
        return torch.from_numpy(oracle.coefficients(Is.float().numpy(), ps.float().numpy(), R,
                                                    eps, 1, oracle.NEAREST))

    def upsample_rows(self, I_own, mean_ext, plan):
        Uy = brute.interp_matrix(plan.H, plan.h)[plan.Y0:plan.Y1, plan.e0:plan.e1]
        Ux = brute.interp_matrix(plan.W, plan.w)
        I = I_own.double().numpy()
        M = mean_ext.double().numpy()
        B, C_I = I.shape[:2]
        C_p = M.shape[1]
        q = np.zeros((B, C_p) + I.shape[2:])
        for b in range(B):
            for c in range(C_p):
                q[b, c] = Uy @ M[b, c, C_I] @ Ux.T
                for j in range(C_I):
                    q[b, c] += (Uy @ M[b, c, j] @ Ux.T) * I[b, j]
        return torch.from_numpy(q)
