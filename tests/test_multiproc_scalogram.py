"""CPU, world_size 2 (gloo): the scalogram's distributed host logic — scale and chunk
sharding, broadcast of the input, point-to-point gather to rank 0 — produces exactly the
single-process result. The per-scale compute is injected (the oracle's restatement of
the reference transform), since this container has no GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_exec(spec, x, begin, count):
    import oracle as O

    c = spec.morlet_coeffs
    full = O.morlet_direct(x.double().numpy(), 1, spec.half_width, spec.beta, spec.n0, spec.alpha,
                           1.0 / (2.0 * spec.sigma ** 2), O.KERNEL_INTEGRAL, O.DOUBLE, c.cos_orders, c.cos_coeffs,
                           c.sin_orders, c.sin_coeffs)
    part = full[begin:begin + count]
    return torch.from_numpy(np.stack([part.real, part.imag], axis=-1).astype(np.float32))


def _worker(rank, world, port, shard, n, sigmas, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_11866_b200 import scalogram as SG

    specs = SG.build_specs(sigmas, xi=8.0, pd=4, threads=2)
    x = torch.zeros(n, dtype=torch.float32)
    if rank == 0:
        import oracle as O

        x = torch.from_numpy(O.make_test_signal(O.SEEDED_NOISE, n, 1234).astype(np.float32))
    dist.broadcast(x, src=0)
    sc = SG.Scalogram(n, specs, world, rank, shard, executor=oracle_exec)
    out = torch.empty((len(sc.rows), sc.count, 2), dtype=torch.float32)
    sc.run(x, out)
    full = sc.gather(out)  # the same point-to-point protocol the NCCL path uses
    ns = len(specs)
    if rank == 0:
        single = SG.Scalogram(n, specs, 1, 0, shard, executor=oracle_exec)
        ref = torch.empty((ns, n, 2), dtype=torch.float32)
        single.run(x, ref)
        q.put(float((full - ref).abs().max()))
    dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["scale", "chunk"])
def test_two_rank_scalogram_matches_single_process(shard):
    from paper_2110_11866_b200 import scalogram as SG

    sigmas = SG.scale_sigmas(5, 8.0, 40.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shard, 2001, sigmas, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=10) == 0.0


def test_sharding_covers_everything_once():
    from paper_2110_11866_b200 import scalogram as SG

    for world in (1, 2, 3, 8):
        rows = sorted(i for r in range(world) for i in SG.shard_scales(128, world, r))
        assert rows == list(range(128))
        spans = [SG.chunk_range(2 ** 24 + 3, world, r) for r in range(world)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == 2 ** 24 + 3
        for (b0, c0), (b1, _) in zip(spans, spans[1:]):
            assert b0 + c0 == b1
    s = SG.scale_sigmas()
    assert len(s) == 128 and abs(s[0] - 16.0) < 1e-12 and abs(s[-1] - 16384.0) < 1e-9
    assert SG.default_n0(16.0) == 4 and SG.default_n0(100.0) == 5
