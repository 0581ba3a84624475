"""Seeded synthetic draft/target distributions of the BASELINE.json shapes (there is no model or dataset here).

Per request b a difficulty is drawn from a two-population mix like MixSource (accept_model.py:134-158): easy requests
(probability `easy_frac`) get a small target-vs-draft logit noise, hard ones a large one.  Draft logits are
N(0,1) with one spiked "mode" token per position (spike height U(spike_lo, spike_hi)), q = softmax(z_q); the target
is p = softmax(z_q + sigma_b * N(0,1)) at the k draft positions and an independent spiked row at the bonus
position.  Draft tokens d ~ q (stochastic) or argmax q (greedy); the selector's confidences are conf = q[b,j,d_bj]
in fp64 (the paper's surrogate).  Uniforms are fp64 in [0,1).  Everything is generated on the device
in row blocks so 17 GB cfg3 tensors never need host memory.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch


@dataclass
class Batch:
    B: int
    k: int
    V: int
    p: torch.Tensor        # [B, k+1, V] f32
    q: torch.Tensor        # [B, k, V] f32
    d: torch.Tensor        # [B, k] i32
    conf: torch.Tensor     # [B, k] f64
    lengths: torch.Tensor  # [B] i32
    u_acc: torch.Tensor    # [B, k] f64
    u_res: torch.Tensor    # [B] f64


def _spiked_softmax_(out: torch.Tensor, g: torch.Generator, spike_lo: float, spike_hi: float,
                     base: Optional[torch.Tensor] = None, sigma: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out[..., V] <- softmax(logits); returns the logits used (for the draft rows, reused by the target)."""
    shape = out.shape
    z = torch.randn(shape, generator=g, device=out.device, dtype=torch.float32)
    if base is None:
        rows = z.view(-1, shape[-1])
        mode = torch.randint(0, shape[-1], (rows.shape[0],), generator=g, device=out.device)
        h = torch.rand(rows.shape[0], generator=g, device=out.device) * (spike_hi - spike_lo) + spike_lo
        rows[torch.arange(rows.shape[0], device=out.device), mode] += h
    else:
        z.mul_(sigma.view(-1, *([1] * (len(shape) - 1)))).add_(base)
    torch.softmax(z, dim=-1, out=out)
    return z


def make_batch(B: int, k: int, V: int, *, mode: str = "stochastic", seed: int = 0, device="cuda",
               ragged: bool = False, easy_frac: float = 0.5, sigma_easy: float = 0.35, sigma_hard: float = 2.0,
               spike_lo: Optional[float] = None, spike_hi: Optional[float] = None,
               block_bytes: int = 1 << 30) -> Batch:
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    import math

    lv = math.log(V)
    spike_lo = lv - 2.0 if spike_lo is None else spike_lo   # draft mode probability ~0.1 ..
    spike_hi = lv + 3.0 if spike_hi is None else spike_hi   # .. ~0.95
    p = torch.empty(B, k + 1, V, dtype=torch.float32, device=dev)
    q = torch.empty(B, k, V, dtype=torch.float32, device=dev)
    easy = torch.rand(B, generator=g, device=dev) < easy_frac
    sigma = torch.where(easy, torch.full((B,), sigma_easy, device=dev), torch.full((B,), sigma_hard, device=dev))
    blk = max(1, int(block_bytes // max(1, (k + 1) * V * 4 * 3)))
    for b0 in range(0, B, blk):
        b1 = min(B, b0 + blk)
        if k > 0:
            zq = _spiked_softmax_(q[b0:b1], g, spike_lo, spike_hi)
            _spiked_softmax_(p[b0:b1, :k], g, spike_lo, spike_hi, base=zq, sigma=sigma[b0:b1])
            del zq
        _spiked_softmax_(p[b0:b1, k:], g, spike_lo, spike_hi)
    if k > 0:
        flat = q.view(-1, V)
        if mode == "greedy":
            d = flat.argmax(dim=-1)
        else:
            d = torch.empty(flat.shape[0], dtype=torch.int64, device=dev)
            rb = max(1, int(block_bytes // (V * 4)))
            for r0 in range(0, flat.shape[0], rb):
                d[r0:r0 + rb] = torch.multinomial(flat[r0:r0 + rb], 1, generator=g).view(-1)
        d = d.view(B, k)
        conf = q.gather(2, d.unsqueeze(-1)).squeeze(-1).to(torch.float64).contiguous()
        d = d.to(torch.int32).contiguous()
    else:
        d = torch.zeros(B, 0, dtype=torch.int32, device=dev)
        conf = torch.zeros(B, 0, dtype=torch.float64, device=dev)
    if ragged and k > 0:
        lengths = torch.randint(1, k + 1, (B,), generator=g, device=dev, dtype=torch.int32)
        full = torch.rand(B, generator=g, device=dev) < 0.5
        lengths = torch.where(full, torch.full_like(lengths, k), lengths)
    else:
        lengths = torch.full((B,), k, dtype=torch.int32, device=dev)
    u_acc = torch.rand(B, k, generator=g, device=dev, dtype=torch.float64)
    u_res = torch.rand(B, generator=g, device=dev, dtype=torch.float64)
    return Batch(B, k, V, p, q, d, conf, lengths, u_acc, u_res)


def selection_instance(B: int, k: int, kind: str, seed: int = 0, device="cuda"):
    """Adversarial selector inputs: 'random', 'quantized' (multiples of 1/64, incl. 0 and 1), 'ties' (one value),
    'zeros' (mostly 0.0 and -0.0), 'ragged' (random lengths).  Returns (alpha [B,k] f64, lengths [B] i32)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    if kind == "quantized":
        a = torch.randint(0, 65, (B, k), generator=g).double() / 64.0
    elif kind == "ties":
        a = torch.full((B, k), 0.5, dtype=torch.float64)
    elif kind == "zeros":
        a = torch.rand(B, k, generator=g, dtype=torch.float64)
        z = torch.rand(B, k, generator=g) < 0.4
        a[z] = 0.0
        nz = torch.rand(B, k, generator=g) < 0.2
        a[nz] = -0.0
    else:
        a = torch.rand(B, k, generator=g, dtype=torch.float64)
    if kind == "ragged":
        lengths = torch.randint(1, k + 1, (B,), generator=g, dtype=torch.int32)
    else:
        lengths = torch.full((B,), k, dtype=torch.int32)
    return a.to(device), lengths.to(device)


@dataclass
class LogitBatch:
    """The same shapes as Batch with the rows as bf16 LOGITS plus their fp32 row log-sum-exp (the logits contract of
    include/tetris_b200.h): zp [B, k+1, V], zq [B, k, V] bf16; lse_p [B, k+1], lse_q [B, k] f32."""
    B: int
    k: int
    V: int
    zp: torch.Tensor
    zq: torch.Tensor
    lse_p: torch.Tensor
    lse_q: torch.Tensor
    d: torch.Tensor
    conf: torch.Tensor
    lengths: torch.Tensor
    u_acc: torch.Tensor
    u_res: torch.Tensor


def make_logit_batch(B: int, k: int, V: int, *, seed: int = 0, device="cuda", ragged: bool = False,
                     easy_frac: float = 0.5, sigma_easy: float = 0.35, sigma_hard: float = 2.0,
                     block_bytes: int = 1 << 30) -> LogitBatch:
    """Spiked draft logits / noisy target logits as in make_batch, stored as bf16; lse = logsumexp of the stored bf16
    values (fp32); draft tokens d ~ softmax(zq); conf = exp(zq[d] - lse_q) in fp64 (the draft's confidence)."""
    import math

    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    lv = math.log(V)
    spike_lo, spike_hi = lv - 2.0, lv + 3.0
    zp = torch.empty(B, k + 1, V, dtype=torch.bfloat16, device=dev)
    zq = torch.empty(B, k, V, dtype=torch.bfloat16, device=dev)
    lse_p = torch.empty(B, k + 1, dtype=torch.float32, device=dev)
    lse_q = torch.empty(B, k, dtype=torch.float32, device=dev)
    d = torch.zeros(B, k, dtype=torch.int64, device=dev)
    easy = torch.rand(B, generator=g, device=dev) < easy_frac
    sigma = torch.where(easy, torch.full((B,), sigma_easy, device=dev), torch.full((B,), sigma_hard, device=dev))
    blk = max(1, int(block_bytes // max(1, (k + 1) * V * 4 * 3)))

    def spiked(n_rows):
        z = torch.randn(n_rows, V, generator=g, device=dev, dtype=torch.float32)
        mode = torch.randint(0, V, (n_rows,), generator=g, device=dev)
        h = torch.rand(n_rows, generator=g, device=dev) * (spike_hi - spike_lo) + spike_lo
        z[torch.arange(n_rows, device=dev), mode] += h
        return z

    for b0 in range(0, B, blk):
        b1 = min(B, b0 + blk)
        nb = b1 - b0
        if k > 0:
            z = spiked(nb * k).view(nb, k, V)
            zq[b0:b1] = z.to(torch.bfloat16)
            zt = z.mul_(0).add_(torch.randn(nb, k, V, generator=g, device=dev)).mul_(sigma[b0:b1].view(-1, 1, 1))
            zt.add_(zq[b0:b1].float())
            zp[b0:b1, :k] = zt.to(torch.bfloat16)
            del z, zt
            lse_q[b0:b1] = torch.logsumexp(zq[b0:b1].float(), dim=-1)
            qprob = torch.softmax(zq[b0:b1].float(), dim=-1).view(-1, V)
            d[b0:b1] = torch.multinomial(qprob, 1, generator=g).view(nb, k)
            del qprob
        zp[b0:b1, k:] = spiked(nb).view(nb, 1, V).to(torch.bfloat16)
        lse_p[b0:b1] = torch.logsumexp(zp[b0:b1].float(), dim=-1)
    if k > 0:
        zd = zq.gather(2, d.unsqueeze(-1)).squeeze(-1).double()
        conf = torch.exp(zd - lse_q.double()).clamp_(0.0, 1.0).contiguous()
    else:
        conf = torch.zeros(B, 0, dtype=torch.float64, device=dev)
    if ragged and k > 0:
        lengths = torch.randint(1, k + 1, (B,), generator=g, device=dev, dtype=torch.int32)
    else:
        lengths = torch.full((B,), k, dtype=torch.int32, device=dev)
    u_acc = torch.rand(B, k, generator=g, device=dev, dtype=torch.float64)
    u_res = torch.rand(B, generator=g, device=dev, dtype=torch.float64)
    return LogitBatch(B, k, V, zp, zq, lse_p, lse_q, d.to(torch.int32).contiguous(), conf, lengths, u_acc, u_res)
