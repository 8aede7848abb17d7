"""GPU parity for K4, the tensor-core chunked transform (csrc/sft_tc.cuh): the same
transforms as K1 (proj/src/transforms.cpp:279-428) evaluated as 3xTF32 tcgen05 GEMMs
over 32-position chunks plus a chunk-state scan. Checked against the fp64 oracle
restatement of the reference combine (north_star: <= 1e-5 relative for fp32 ASFT), and
row by row against K1 (the CUDA-core kernel) on the same inputs."""
import numpy as np
import pytest

from conftest import rel_max
from test_gpu_transforms import oracle_transform

pytestmark = pytest.mark.gpu


def _run(sft, spec, xb, mode, boundary=1, out_range=None):
    import torch

    n = xb.shape[1]
    plan = sft.TransformPlan(spec, n, xb.shape[0], boundary, out_range, mode=mode)
    out = plan.empty_output()
    plan.execute(xb, out)
    torch.cuda.synchronize()
    oh = out.double().cpu().numpy()
    return plan, (oh[..., 0] + 1j * oh[..., 1] if plan.complex_out else oh)


CASES = [
    # abbreviation, sigma, xi, n, batch
    ("MMS5P3", 8192.0, 10.0, 102400, 6),   # BASELINE config 4 shape (2P+1 = 7 orders, complex injection)
    ("MDS5P6", 8192.0, 10.0, 102400, 2),   # config 3 spec (6 orders, real injection)
    ("GDS10P6", 8192.0, 0.0, 102400, 2),   # config 2 spec, real output
    ("MDS3P6", 40.0, 8.0, 20001, 3),       # small sigma, partial last tile
    ("MMS2P3", 64.0, 10.0, 9000, 5),
    ("GDS4P5", 512.0, 0.0, 50000, 2),
    ("MDP6", 1000.0, 10.0, 30000, 2),      # SFT (alpha = 0)
    ("GDP6", 4000.0, 0.0, 102400, 2),      # Gaussian SFT, real output
    ("MMS1P2", 20.0, 12.0, 40000, 7),      # tiny sigma: one warm-up tile
]


@pytest.mark.parametrize("abbrev,sigma,xi,n,batch", CASES)
def test_tc_vs_oracle_and_cuda_core(sft, O, abbrev, sigma, xi, n, batch):
    spec = sft.make_transform_spec(abbrev, sigma, xi, sft.TransformOptions(precision=0))
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 77, batch, sft.Precision.Single)
    plan, tc = _run(sft, spec, xb, "tc")
    assert plan.describe()["tensor_cores"] == 1
    _, ref1 = _run(sft, spec, xb, "seq")
    xh = xb.double().cpu().numpy()
    for b in sorted({0, batch - 1}):
        assert rel_max(tc[b], oracle_transform(O, xh[b], 1, spec)) < 1e-5
    assert rel_max(tc, ref1) < 1e-5


@pytest.mark.parametrize("gkind,n0", [(1, 0), (1, 5), (2, 0), (2, 5)])
def test_tc_gaussian_derivatives(sft, O, gkind, n0):
    """First / second Gaussian derivatives (proj/src/transforms.cpp:279-335 weights on the
    sin / cos components, plus the ASFT corrections for n0 > 0) on K4."""
    spec = sft.make_gauss_spec(700.0, gkind, 6, n0, sft.TransformOptions(precision=0))
    n, batch = 40000, 2
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 13, batch, sft.Precision.Single)
    _, tc = _run(sft, spec, xb, "tc")
    _, k1 = _run(sft, spec, xb, "seq")
    xh = xb.double().cpu().numpy()
    assert rel_max(tc[1], oracle_transform(O, xh[1], 1, spec)) < 1e-5
    assert rel_max(tc, k1) < 1e-5


@pytest.mark.parametrize("boundary", [0, 1])
def test_tc_boundaries_and_offset(sft, O, boundary):
    """Both boundary policies, and a DC offset (x + 1, the fp32 cancellation case)."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 300.0, 10.0, sft.TransformOptions(precision=0))
    n = 12345
    x = O.make_test_signal(O.SEEDED_NOISE, n, 5) + 1.0
    xb = torch.tensor(np.stack([x, -x]), dtype=torch.float32, device="cuda")
    _, tc = _run(sft, spec, xb, "tc", boundary)
    xh = xb.double().cpu().numpy()
    for b in range(2):
        assert rel_max(tc[b], oracle_transform(O, xh[b], boundary, spec)) < 1e-5


@pytest.mark.parametrize("boundary", [0, 1])
def test_tc_skipped_constant_warmup(sft, O, boundary):
    """Config-4 geometry (sigma = 8192, n0 = 5): six leading warm-up tiles of every signal
    read only boundary samples and are replaced by their closed-form state; both boundary
    policies, and a DC offset so the clamped boundary value is far from zero (x + 1: larger
    offsets are ill-conditioned in fp32 for every kernel, K1 included, tools/dc_probe.py)."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 8192.0, 10.0, sft.TransformOptions(precision=0))
    n = 102400
    x = O.make_test_signal(O.SEEDED_NOISE, n, 11) + 1.0
    xb = torch.tensor(np.stack([x, 0.5 * x]), dtype=torch.float32, device="cuda")
    _, tc = _run(sft, spec, xb, "tc", boundary)
    xh = xb.double().cpu().numpy()
    for b in range(2):
        assert rel_max(tc[b], oracle_transform(O, xh[b], boundary, spec)) < 1e-5


def test_tc_ranged_plan_matches_full(sft, O):
    """Output-range plans (chunk sharding with halo) reproduce the full transform. The two
    are different fp32 evaluations of the same sums (the range plan warms up from its own
    window start), so they agree to fp32 rounding; each is checked against the fp64
    oracle at the north_star bound."""
    spec = sft.make_transform_spec("MDS5P6", 2000.0, 10.0, sft.TransformOptions(precision=0))
    n = 60000
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 3, 1, sft.Precision.Single)
    _, full = _run(sft, spec, xb, "tc")
    ref = oracle_transform(O, xb[0].double().cpu().numpy(), 1, spec)
    assert rel_max(full[0], ref) < 1e-5
    for b, c in ((0, 7000), (23456, 20000), (n - 9999, 9999)):
        _, part = _run(sft, spec, xb, "tc", 1, (b, c))
        assert rel_max(part[0], full[0, b:b + c]) < 5e-6
        assert rel_max(part[0], ref[b:b + c]) < 1e-5


def test_tc_selection(sft, O):
    """Auto mode picks K4 for eligible transforms spanning >= 4 x 148 tiles (config 4)."""
    spec = sft.make_transform_spec("MMS5P3", 8192.0, 10.0, sft.TransformOptions(precision=0))
    assert sft.TransformPlan(spec, 102400, 4096).describe()["tensor_cores"] == 1
    assert sft.TransformPlan(spec, 102400, 1).describe()["tensor_cores"] == 0
    fp64 = sft.make_transform_spec("MMS5P3", 8192.0, 10.0, sft.TransformOptions(precision=1))
    assert sft.TransformPlan(fp64, 102400, 4096).describe()["tensor_cores"] == 0


def test_tc_rejects_ineligible_specs(sft):
    fp64 = sft.make_transform_spec("MDS5P6", 100.0, 10.0, sft.TransformOptions(precision=1))
    with pytest.raises(ValueError):
        sft.TransformPlan(fp64, 10000, 2, mode="tc")


def test_tc_strided_and_unaligned_outputs(sft, O):
    """Output layouts the TMA store cannot take: a padded row stride with count % 32 != 0,
    and a row base offset by one complex element (8 bytes): K4 falls back to 16-byte /
    element stores and matches the packed TMA result."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 600.0, 10.0, sft.TransformOptions(precision=0))
    n, B = 30001, 3
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 21, B, sft.Precision.Single)
    plan = sft.TransformPlan(spec, n, B, mode="tc")
    ref = plan.empty_output()
    plan.execute(xb, ref)
    ld = n + 7
    big = torch.full((B * ld + 1, 2), float("nan"), dtype=torch.float32, device="cuda")
    for off in (0, 1):
        big.fill_(float("nan"))
        view = big[off:off + B * ld].view(B, ld, 2)
        plan.execute(xb, view, ld_out=ld)
        torch.cuda.synchronize()
        assert torch.equal(view[:, :n], ref)
        assert torch.isnan(view[:, n:]).all()  # nothing written past count


def test_tc_long_signal_chunks_match_cuda_core(sft, O):
    """One long signal split into chunk items across the persistent CTAs (each chunk with
    its own warm-up) equals K1's sequential result; first/last samples vs the oracle."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 3000.0, 10.0, sft.TransformOptions(precision=0))
    n = 1 << 21
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 5, 1, sft.Precision.Single)
    plan, tc = _run(sft, spec, xb, "tc")
    assert plan.describe()["chunks_per_signal"] > 1
    _, k1 = _run(sft, spec, xb, "seq")
    assert rel_max(tc, k1) < 1e-5
    head = xb[0, :40000].double().cpu().numpy()
    ref = oracle_transform(O, head, 1, spec)
    # outputs far enough from the cut end are independent of the truncation
    m = 40000 - 3 * 9100
    assert rel_max(tc[0, :m], ref[:m]) < 1e-5


def test_tc_batch_smaller_than_sms(sft, O):
    """A few long signals, each cut into fixed chunks (at most max(256, 16 W) output tiles,
    each with its own warm-up) spread over the persistent CTAs; the cut depends on the
    spec and the length only, so every signal's result is bit-identical whether it runs
    in a batch or alone."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 1000.0, 10.0, sft.TransformOptions(precision=0))
    n, B = 1200000, 3
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 8, B, sft.Precision.Single)
    plan, tc = _run(sft, spec, xb, "tc")
    assert plan.describe()["chunks_per_signal"] == 2
    _, k1 = _run(sft, spec, xb, "seq")
    assert rel_max(tc, k1) < 1e-5
    _, alone = _run(sft, spec, xb[1:2].contiguous(), "tc")
    assert np.array_equal(alone[0], tc[1])


def test_tc_subbatched_host_execution(sft, O):
    """sftgpu_transform_execute_host on a large K4 plan pipelines sub-batches of signals
    through two device staging slots (H2D / kernel / D2H overlap): the result equals the
    device-buffer execution bit for bit."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 300.0, 10.0, sft.TransformOptions(precision=0))
    n, B = 102400, 250  # 307 MB of host input + output: above the sub-batching threshold
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 17, B, sft.Precision.Single)
    plan = sft.TransformPlan(spec, n, B)
    assert plan.describe()["tensor_cores"] == 1
    ref = plan.empty_output()
    plan.execute(xb, ref)
    torch.cuda.synchronize()
    xh = xb.cpu().numpy()
    oh = np.empty(tuple(ref.shape), dtype=np.float32)
    plan.execute_host(xh, oh)
    assert np.array_equal(oh, ref.cpu().numpy())


@pytest.mark.parametrize("offset,pad", [(1, 3), (0, 5), (2, 0)])
def test_tc_unaligned_input(sft, O, offset, pad):
    """Input rows that are not 16-byte aligned (base offset, odd leading dimension): K4's
    loader cannot use TMA boxes or 16-byte copies and stages every stream per sample
    (csrc/sft_tc.cuh, kMixed); results must match the aligned run bit for bit."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 600.0, 10.0, sft.TransformOptions(precision=0))
    n, batch = 30000, 3
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 21, batch, sft.Precision.Single)
    plan = sft.TransformPlan(spec, n, batch, mode="tc")
    ref = plan.empty_output()
    plan.execute(xb, ref)
    ld = n + pad
    buf = torch.zeros(offset + batch * ld, dtype=torch.float32, device="cuda")
    view = buf[offset:offset + batch * ld].view(batch, ld)
    view[:, :n] = xb
    out = plan.empty_output()
    plan.execute(buf[offset:], out, ld_x=ld)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    xh = xb.double().cpu().numpy()
    got = out.double().cpu().numpy()
    assert rel_max(got[1, :, 0] + 1j * got[1, :, 1], oracle_transform(O, xh[1], 1, spec)) < 1e-5


@pytest.mark.parametrize("n,out_range", [(300000, None), (1 << 21, None), (1 << 21, (700001, 500000))])
def test_multiscale_plan_matches_per_scale(sft, O, n, out_range):
    """One persistent multi-scale K4 launch over several scales of one signal (config 5's
    shape, sftgpu_multiscale_plan_create) equals the per-scale plans bit for bit (same
    fixed chunking per spec; scale switches reload the operand image mid-CTA), and the
    fp64 oracle on a window."""
    import torch
    from paper_2110_11866_b200 import scalogram as SG

    sigmas = [16.0, 90.0, 700.0, 2500.0, 6000.0]
    specs = SG.build_specs(sigmas, 10.0, 6)
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 99, 1, sft.Precision.Single)[0]
    plan = sft.MultiScalePlan(specs, n, 1, out_range)
    assert plan.describe()["tensor_cores"] == 1 and plan.batch == len(specs)
    out = plan.empty_output()
    plan.execute(x, out)
    for s, sp in enumerate(specs):
        p1 = sft.TransformPlan(sp, n, 1, 1, out_range, mode="tc")
        o1 = p1.empty_output()
        p1.execute(x, o1)
        torch.cuda.synchronize()
        assert torch.equal(out[s], o1[0]), f"scale {s}"
    b = out_range[0] if out_range else 0
    head = x[:b + 60000].double().cpu().numpy()
    oh = out.double().cpu().numpy()
    for s in (0, 3):
        ref = oracle_transform(O, head, 1, specs[s])[b:b + 30000]
        assert rel_max(oh[s, :30000, 0] + 1j * oh[s, :30000, 1], ref) < 1e-5


def test_multiscale_plan_rejects_mixed_specs(sft):
    from paper_2110_11866_b200 import scalogram as SG

    specs = SG.build_specs([50.0, 400.0], 10.0, 6)
    gd = sft.make_gauss_spec(100.0, sft.GaussKind.Value, 6, 2, sft.TransformOptions(precision=0))
    with pytest.raises(ValueError):
        sft.MultiScalePlan([specs[0], gd], 100000)
    f64 = sft.make_transform_spec("MDS2P6", 50.0, 10.0, sft.TransformOptions(precision=1))
    with pytest.raises(ValueError):
        sft.MultiScalePlan([f64], 100000)
