"""Multi-scale Morlet scalogram (BASELINE config 5) and its multi-GPU sharding.

One Morlet-direct transform per scale sigma_i (ASFT, n0 = min(5, floor(sigma/4)),
P_S auto-selected per scale, fp32), all over the same signal. Work is partitioned
across ranks (one process per GPU) without any cross-GPU carry:

* ``shard="scale"``: rank r owns scales i with i % world == r and computes them over
  the whole signal (the default: every scale is an independent transform);
* ``shard="chunk"``: rank r owns output range [r*N/W, (r+1)*N/W) of every scale; each
  plan reads its window halo (K + n0 samples on both sides, boundary policy at the
  signal ends) straight from the broadcast input, so no scan carry crosses GPUs.

Collectives: the input is broadcast once before any transform runs; the optional
final gather to rank 0 is point-to-point (NCCL has no gather), timed separately.
The kernels are the product ones: one persistent multi-scale K4 launch per <= 128 scales
(``MultiScalePlan``), else per-scale ``TransformPlan``s; the ``executor`` hook exists so the distributed host logic can be exercised on CPU
(gloo) with a checker in tests.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

from . import sft as S


def scale_sigmas(n_scales: int = 128, smin: float = 16.0, smax: float = 16384.0) -> list[float]:
    """sigma_i = smin * (smax/smin)^(i/(n-1))."""
    if n_scales == 1:
        return [smin]
    return [smin * (smax / smin) ** (i / (n_scales - 1)) for i in range(n_scales)]


def default_n0(sigma: float) -> int:
    return min(5, int(math.floor(sigma / 4.0)))


def shard_scales(n_scales: int, world: int, rank: int) -> list[int]:
    """Interleaved assignment: neighbouring scales (similar cost) land on different ranks."""
    return [i for i in range(n_scales) if i % world == rank]


def chunk_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous output range of rank r: [begin, begin + count)."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def build_specs(sigmas, xi: float = 10.0, pd: int = 6, precision=S.Precision.Single, cache: str | None = None,
                threads: int | None = None):
    """Fit (or load) one MorletDirect spec per scale. Fits run in parallel host threads
    (ctypes releases the GIL); ``cache`` is an "sft-coefficients v1" file reused when its
    sets match (sigma, xi, n0, P_D)."""
    if cache and os.path.exists(cache):
        try:
            sets = S.read_coefficient_sets(cache)
            ok = len(sets) == len(sigmas) and all(
                abs(s.sigma - sg) <= 1e-9 * sg and s.xi == xi and s.n0 == default_n0(sg) and s.n_cos == pd
                for s, sg in zip(sets, sigmas))
            if ok:
                return [S.morlet_direct_spec_from_coeffs(s, precision, S.Strategy.KernelIntegral, False) for s in sets]
        except (ValueError, OSError):
            pass
    opts = S.TransformOptions(precision=precision, strategy=S.Strategy.KernelIntegral)

    def fit(sg):
        return S.make_morlet_direct_spec(sg, xi, pd, default_n0(sg), opts)

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 4) as ex:
        specs = list(ex.map(fit, sigmas))
    if cache:
        try:
            S.write_coefficient_sets(cache, specs)
        except (ValueError, OSError):
            pass
    return specs


class Scalogram:
    """Rank-local part of a scalogram: ``rows`` scales x ``count`` outputs (complex)."""

    def __init__(self, n: int, specs, world: int = 1, rank: int = 0, shard: str = "scale",
                 boundary=S.BoundaryPolicy.Clamp, executor=None, streams: int = 8, mode: str = "auto"):
        if shard not in ("scale", "chunk"):
            raise ValueError("shard must be 'scale' or 'chunk'")
        self.n, self.specs, self.world, self.rank, self.shard = n, list(specs), world, rank, shard
        self.boundary = boundary
        if shard == "scale":
            self.rows = shard_scales(len(self.specs), world, rank)
            self.begin, self.count = 0, n
        else:
            self.rows = list(range(len(self.specs)))
            self.begin, self.count = chunk_range(n, world, rank)
        self.executor = executor
        self.plans = []
        self.n_streams = streams
        self._streams = None
        self.multi = []  # (first row, MultiScalePlan over rows [first, first + plan.batch))
        if executor is None:
            # mode "auto": the rank's scales in persistent multi-scale tensor-core launches
            # (K4 over every scale's fixed chunks, <= 128 scales each) when every spec
            # qualifies; otherwise one plan per scale: K4 where the scale qualifies, else
            # sequential K1 plans (chunked, few CTAs each, so scales run concurrently on
            # several streams with no inter-CTA look-back)
            rng = (self.begin, self.count)
            if mode == "auto":
                try:
                    for r0 in range(0, len(self.rows), 128):
                        sub = [self.specs[i] for i in self.rows[r0:r0 + 128]]
                        self.multi.append((r0, S.MultiScalePlan(sub, n, boundary, rng)))
                except ValueError:
                    self.multi = []
            if not self.multi:
                for i in self.rows:
                    p = S.TransformPlan(self.specs[i], n, 1, boundary, rng, mode=mode)
                    if mode == "auto" and not p.describe()["tensor_cores"]:
                        p = S.TransformPlan(self.specs[i], n, 1, boundary, rng, mode="seq")
                    self.plans.append(p)

    @property
    def launches(self) -> int:
        return sum(p.launches for p in self.plans) + sum(p.launches for _, p in self.multi)

    def output_bytes(self, itemsize: int = 4) -> int:
        return len(self.rows) * self.count * 2 * itemsize

    def empty_output(self):
        import torch

        return torch.empty((len(self.rows), self.count, 2), dtype=torch.float32, device="cuda")

    def run(self, x, out):
        """x: the full signal (device tensor, fp32); out: [rows][count][2]."""
        if self.executor is not None:
            for r, i in enumerate(self.rows):
                out[r] = self.executor(self.specs[i], x, self.begin, self.count)
            return out
        import torch

        if self.multi:
            for r0, p in self.multi:
                p.execute(x, out[r0:r0 + p.batch])
            return out
        cur = torch.cuda.current_stream()
        if self._streams is None:
            self._streams = [torch.cuda.Stream() for _ in range(self.n_streams)]
        ev = torch.cuda.Event()
        ev.record(cur)
        for s_ in self._streams:
            s_.wait_event(ev)
        # largest scales (longest warm-up, fewest chunks) first, spread over the streams
        order = sorted(range(len(self.plans)), key=lambda r: -self.specs[self.rows[r]].half_width)
        for j, r in enumerate(order):
            s_ = self._streams[j % self.n_streams]
            with torch.cuda.stream(s_):
                self.plans[r].execute(x, out[r], stream=s_.cuda_stream)
        for s_ in self._streams:
            e = torch.cuda.Event()
            e.record(s_)
            cur.wait_event(e)
        return out

    def gather(self, out, group=None):
        """Assembles the full [n_scales][n][2] scalogram on rank 0 (point-to-point)."""
        import torch
        import torch.distributed as dist

        ns = len(self.specs)
        if self.world == 1:
            return out
        full = None
        if self.rank == 0:
            full = torch.empty((ns, self.n, 2), dtype=out.dtype, device=out.device)
            self._place(full, out, 0)
            for src in range(1, self.world):
                rows, (b, c) = self._layout(src)
                buf = torch.empty((len(rows), c, 2), dtype=out.dtype, device=out.device)
                dist.recv(buf, src=src, group=group)
                self._place(full, buf, src)
        else:
            dist.send(out.contiguous(), dst=0, group=group)
        return full

    def _layout(self, rank):
        if self.shard == "scale":
            return shard_scales(len(self.specs), self.world, rank), (0, self.n)
        return list(range(len(self.specs))), chunk_range(self.n, self.world, rank)

    def _place(self, full, part, rank):
        rows, (b, c) = self._layout(rank)
        for r, i in enumerate(rows):
            full[i, b:b + c] = part[r]


def scalogram_bytes(n: int, n_scales: int) -> int:
    """Algorithmic bytes of one scalogram: fp32 input read once per scale pass + complex64 out."""
    return n_scales * n * (4 + 8)


__all__ = ["scale_sigmas", "default_n0", "shard_scales", "chunk_range", "build_specs", "Scalogram",
           "scalogram_bytes"]
