"""GPU, world size 2 on one device (gloo for the host-side collectives, both ranks on
cuda:0): the scalogram's distributed path with the REAL kernels (persistent multi-scale
K4 launches, csrc/sft_tc.cuh) in both shardings. Scale sharding reproduces the
single-process GPU result bit for bit (every scale is computed whole on its rank, with
the same fixed chunking); chunk sharding (each rank an output range of every scale, its
K + n0 halo read from the broadcast input) agrees to fp32 rounding, and both match the
fp64 oracle on a window (north_star: <= 1e-5 relative)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SIGMAS = [16.0, 60.0, 250.0, 900.0, 3000.0]
N = 1 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shard, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2110_11866_b200 as P
    from paper_2110_11866_b200 import scalogram as SG

    specs = SG.build_specs(SIGMAS, xi=10.0, pd=6, threads=4)
    xc = torch.zeros(N, dtype=torch.float32)
    if rank == 0:
        xc = P.generate_signals(P.TestSignalKind.SeededNoise, N, 4321, 1, P.Precision.Single)[0].cpu()
    dist.broadcast(xc, src=0)  # input broadcast once (the NCCL path broadcasts on device)
    x = xc.cuda()
    sc = SG.Scalogram(N, specs, world, rank, shard)
    assert sc.multi, "expected the multi-scale K4 path"
    out = sc.empty_output()
    sc.run(x, out)
    torch.cuda.synchronize()
    full = sc.gather(out.cpu())  # point-to-point to rank 0, same protocol as with NCCL
    if rank == 0:
        q.put(full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["scale", "chunk"])
def test_two_ranks_real_kernels(shard, O):
    import paper_2110_11866_b200 as P
    from conftest import rel_max
    from paper_2110_11866_b200 import scalogram as SG
    from test_gpu_transforms import oracle_transform

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shard, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    specs = SG.build_specs(SIGMAS, xi=10.0, pd=6, threads=4)
    x = P.generate_signals(P.TestSignalKind.SeededNoise, N, 4321, 1, P.Precision.Single)[0]
    single = SG.Scalogram(N, specs)
    ref = single.empty_output()
    single.run(x, ref)
    ref = ref.cpu().numpy()
    if shard == "scale":
        assert np.array_equal(got, ref)
    else:
        for s in range(len(specs)):
            assert rel_max(got[s, :, 0] + 1j * got[s, :, 1], ref[s, :, 0] + 1j * ref[s, :, 1]) < 5e-6
    # the halo boundary of the chunk split (N/2) and the head, against the fp64 oracle
    xh = x.double().cpu().numpy()
    for s in (1, 3):
        w0 = N // 2 - 20000
        seg = oracle_transform(O, xh, 1, specs[s])[w0:w0 + 40000]
        assert rel_max(got[s, w0:w0 + 40000, 0] + 1j * got[s, w0:w0 + 40000, 1], seg) < 1e-5
