"""Row-band decomposition of one large image across ranks.

Rank k owns low-res rows [y0, y1) = [k h // G, (k+1) h // G) of the h = ceil(H/s) low-res
rows, i.e. full-resolution rows [y0 s, min(H, y1 s)) (band edges on multiples of s, so the
subsample grid is the global one, R3/R4).  Its own full-resolution rows upsample from low-res
rows [y0 - 1, y1] (R5), whose mean_a, mean_b need a, b on rows +-r' further and those need
I', p' on rows +-r' further again, so a single exchange of HALO = 2r' + 1 low-res rows of I'
and p' with each neighbour makes everything after it local (the "single-step" variant of
SURVEY §8(e)).  Windows clip at the global image bounds because the extended band is clipped
to [0, h): at interior band edges the clipped windows only affect a, b rows the rank never
uses.  Stages (all in libfgf.so kernels):

    fgf_subsample (own rows) -> exchange halos -> fgf_lowres_mean (extended band)
    -> fgf_upsample_output_rows (own rows, global vertical map)

The exchange is an object with `exchange(send_up, send_down) -> (from_up, from_down)`:
`DistExchange` uses torch.distributed point-to-point (NCCL over NVLink on GPUs, gloo on CPU);
single-process simulations pass the neighbours' planes directly (`filter_bands_local`).
The compute backend is pluggable so the host logic can be tested on CPU against the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass


def lowres_radius(r: int, s: int) -> int:
    """R2: r' = max(1, floor(r/s + 1/2)) -- from the C planner (fgf_band_geometry)."""
    from paper_1505_00996_b200 import fgf_band_geometry
    return fgf_band_geometry(max(1, s), 1, r, s, 1, 0)[2]


@dataclass(frozen=True)
class BandPlan:
    H: int
    W: int
    s: int
    r: int
    world: int
    rank: int
    h: int
    w: int
    R: int          # r'
    halo: int       # 2 r' + 1 low-res rows
    y0: int         # own low-res rows [y0, y1)
    y1: int
    Y0: int         # own full-res rows [Y0, Y1)
    Y1: int
    e0: int         # extended low-res rows [e0, e1) after the exchange
    e1: int


def plan_band(H: int, W: int, r: int, s: int, world: int, rank: int) -> BandPlan:
    """The band of `rank`, from the C planner of libfgf.so (fgf_band_geometry: one rule for the
    C band path and this one; host logic only, no GPU needed)."""
    from paper_1505_00996_b200 import FGF_ERR_PARAM, FGFError, fgf_band_geometry
    try:
        h, w, R, halo, y0, y1, Y0, Y1, e0, e1 = fgf_band_geometry(H, W, r, s, world, rank)
    except FGFError as e:
        if e.status == FGF_ERR_PARAM:
            raise ValueError(f"bands of {-(-H // s) // world} low-res rows are thinner than the "
                             "halo (2r'+1 rows): use fewer ranks") from e
        raise
    return BandPlan(H, W, s, r, world, rank, h, w, R, halo, y0, y1, Y0, Y1, e0, e1)


class DistExchange:
    """Halo exchange with the rank's neighbours over torch.distributed P2P."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, send_up, send_down):
        import torch
        import torch.distributed as dist
        ops, from_up, from_down = [], None, None
        if self.rank > 0:
            from_up = torch.empty_like(send_up)
            ops.append(dist.P2POp(dist.isend, send_up.contiguous(), self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, from_up, self.rank - 1, self.group))
        if self.rank < self.world - 1:
            from_down = torch.empty_like(send_down)
            ops.append(dist.P2POp(dist.isend, send_down.contiguous(), self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, from_down, self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return from_up, from_down


class GpuBackend:
    """The three stages through the C ABI (libfgf.so) on CUDA tensors."""

    def __init__(self, stream=None):
        self.stream = stream
        self.ws = None

    def subsample(self, x, s, sub_mode):
        import torch

        import paper_1505_00996_b200 as fgf
        B, C, H, W = x.shape
        out = torch.empty((B, C, -(-H // s), -(-W // s)), dtype=x.dtype, device=x.device)
        fgf.fgf_subsample(x, out, B * C, H, W, s, sub_mode, stream=self._st(x))
        return out

    def lowres_mean(self, Is, ps, R, eps):
        import torch

        import paper_1505_00996_b200 as fgf
        B, C_I, h, w = Is.shape
        C_p = ps.shape[1]
        mean = torch.empty((B, C_p, C_I + 1, h, w), dtype=Is.dtype, device=Is.device)
        nb = fgf.fgf_lowres_workspace_bytes(B, h, w, C_I, C_p)
        if self.ws is None or self.ws.numel() < nb:
            self.ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=Is.device)
        fgf.fgf_lowres_mean(Is, ps, mean, B, h, w, C_I, C_p, R, eps, self.ws, self.ws.numel(),
                            stream=self._st(Is))
        return mean

    def upsample_rows(self, I_own, mean_ext, plan: BandPlan):
        import torch

        import paper_1505_00996_b200 as fgf
        B, C_I, rows, W = I_own.shape
        C_p = mean_ext.shape[1]
        q = torch.empty((B, C_p, rows, W), dtype=I_own.dtype, device=I_own.device)
        fgf.fgf_upsample_output_rows(I_own, mean_ext, q, B, rows, W, C_I, C_p, plan.H, plan.h,
                                     plan.w, plan.Y0, plan.e0, plan.e1 - plan.e0,
                                     stream=self._st(I_own))
        return q

    def _st(self, t):
        import torch
        return self.stream if self.stream is not None else torch.cuda.current_stream(t.device)


def _own_lowres(I_own, p_own, plan: BandPlan, sub_mode, backend):
    Is = backend.subsample(I_own, plan.s, sub_mode)
    ps = Is if p_own is I_own else backend.subsample(p_own, plan.s, sub_mode)
    return Is, ps


def _extend(own, from_up, from_down, plan: BandPlan):
    import torch
    parts = []
    if from_up is not None:
        parts.append(from_up[:, :, from_up.shape[2] - (plan.y0 - plan.e0):])
    parts.append(own)
    if from_down is not None:
        parts.append(from_down[:, :, :plan.e1 - plan.y1])
    return torch.cat(parts, dim=2).contiguous() if len(parts) > 1 else own


def filter_band(I_own, p_own, r, eps, s, sub_mode, H, rank, world, exchange, backend=None):
    """q for this rank's own rows.  I_own, p_own: [B, C, Y1 - Y0, W] (p_own may be I_own)."""
    import torch
    backend = backend or GpuBackend()
    W = I_own.shape[3]
    plan = plan_band(H, W, r, s, world, rank)
    if I_own.shape[2] != plan.Y1 - plan.Y0:
        raise ValueError(f"rank {rank} owns rows [{plan.Y0}, {plan.Y1}) but got {I_own.shape[2]}")
    Is, ps = _own_lowres(I_own, p_own, plan, sub_mode, backend)
    both = Is if ps is Is else torch.cat([Is, ps], dim=1)
    h_own = plan.y1 - plan.y0
    send_up = both[:, :, :min(plan.halo, h_own)]
    send_down = both[:, :, max(0, h_own - plan.halo):]
    from_up, from_down = exchange.exchange(send_up, send_down) if world > 1 else (None, None)
    ext = _extend(both, from_up, from_down, plan)
    C_I = I_own.shape[1]
    Is_e = ext if ps is Is else ext[:, :C_I].contiguous()
    ps_e = Is_e if ps is Is else ext[:, C_I:].contiguous()
    mean = backend.lowres_mean(Is_e, ps_e, plan.R, eps)
    return backend.upsample_rows(I_own, mean, plan)


def filter_bands_local(I, p, r, eps, s, sub_mode, world, backend=None):
    """Single-process simulation of `world` ranks (neighbours' planes passed directly, no
    collective): the test double of the multi-GPU band path.  Returns the stitched q."""
    import torch
    backend = backend or GpuBackend()
    B, C_I, H, W = I.shape
    plans = [plan_band(H, W, r, s, world, k) for k in range(world)]
    own = []
    for pl in plans:
        Io = I[:, :, pl.Y0:pl.Y1].contiguous()
        po = Io if p is I else p[:, :, pl.Y0:pl.Y1].contiguous()
        Is, ps = _own_lowres(Io, po, pl, sub_mode, backend)
        own.append((Io, po, Is if ps is Is else torch.cat([Is, ps], dim=1), ps is Is))
    out = []
    for k, pl in enumerate(plans):
        Io, po, both, self_guided = own[k]
        up = own[k - 1][2][:, :, -pl.halo:] if k > 0 else None
        down = own[k + 1][2][:, :, :pl.halo] if k < world - 1 else None
        ext = _extend(both, up, down, pl)
        Is_e = ext if self_guided else ext[:, :C_I].contiguous()
        ps_e = Is_e if self_guided else ext[:, C_I:].contiguous()
        mean = backend.lowres_mean(Is_e, ps_e, pl.R, eps)
        out.append(backend.upsample_rows(Io, mean, pl))
    return torch.cat(out, dim=2)
