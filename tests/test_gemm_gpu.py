"""K1 (FP32 SIMT) parity on the B200 through the C-ABI.

Every config must be bit-identical (value equality) to the sequential-fmaf
oracle (oracle/gemm_ref.c) -- the kernel accumulates each C element in
increasing k with fmaf from +0 -- and within rel-Frobenius 1e-5 of the
float64 matmul (BASELINE config 1, north_star tolerance).
"""

import numpy as np
import pytest

from oracle.gemm_oracle import gemm_f32_exact, gemm_f64

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _gemm():
    from paper_2003_06795_b200 import gemm
    return gemm


def _dataset():
    from paper_2003_06795_b200 import dataset
    return dataset


def _operands(rng, m, k, n, ta, tb):
    a_store = rng.uniform(-1, 1, size=(k, m) if ta else (m, k)).astype(np.float32)
    b_store = rng.uniform(-1, 1, size=(n, k) if tb else (k, n)).astype(np.float32)
    a = torch.from_numpy(a_store).cuda()
    b = torch.from_numpy(b_store).cuda()
    return a_store, b_store, (a.t() if ta else a), (b.t() if tb else b)


def _run(cfg, m, k, n, ta=False, tb=False, seed=0):
    rng = np.random.default_rng(seed)
    a_store, b_store, a, b = _operands(rng, m, k, n, ta, tb)
    got = _gemm().matmul(a, b, cfg).cpu().numpy()
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta, trans_b=tb).reshape(m, n)
    return got, want, a_store, b_store


def test_baseline_config1_256_cubed():
    """BASELINE configs[0]: 256^3, tile 4x4, acc 4, work-group 8x8."""
    ds = _dataset()
    cfg = ds.KernelConfig(4, 4, 4, 8, 8)
    assert ds.all_configs().index(cfg) == 422
    got, want, a, b = _run(cfg, 256, 256, 256)
    np.testing.assert_array_equal(got, want)
    ref = gemm_f64(a, b)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-5, rel


@pytest.mark.parametrize("shape", [(17, 27, 15), (33, 64, 70)])
def test_every_config_bit_exact_nn(shape):
    m, k, n = shape
    rng = np.random.default_rng(1)
    a_store, b_store, a, b = _operands(rng, m, k, n, False, False)
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n).reshape(m, n)
    bad = []
    for cfg in _dataset().all_configs():
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(cfg.as_tuple())
    assert not bad, f"{len(bad)} configs differ, first {bad[:5]}"


@pytest.mark.parametrize("ta,tb", [(False, True), (True, False), (True, True)])
def test_every_config_bit_exact_transposed(ta, tb):
    m, k, n = 37, 45, 29
    rng = np.random.default_rng(2)
    a_store, b_store, a, b = _operands(rng, m, k, n, ta, tb)
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta,
                          trans_b=tb).reshape(m, n)
    bad = []
    for cfg in _dataset().all_configs():
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(cfg.as_tuple())
    assert not bad, f"{len(bad)} configs differ, first {bad[:5]}"


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 7, 1), (2049, 17, 3), (3, 2049, 5),
                                   (64, 64, 64), (128, 96, 160)])
@pytest.mark.parametrize("cfg", [(1, 1, 1, 1, 64), (8, 8, 8, 16, 16), (2, 8, 1, 128, 1),
                                 (4, 1, 8, 1, 128), (8, 4, 2, 32, 8)])
def test_edge_shapes(shape, cfg):
    ds = _dataset()
    for ta in (False, True):
        for tb in (False, True):
            got, want, _, _ = _run(ds.KernelConfig(*cfg), *shape, ta=ta, tb=tb, seed=3)
            np.testing.assert_array_equal(got, want)


def test_strided_batched_alpha_beta():
    ds = _dataset()
    rng = np.random.default_rng(4)
    batch, m, k, n = 3, 40, 24, 36
    a = rng.uniform(-1, 1, (batch, m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (batch, k, n)).astype(np.float32)
    c0 = rng.uniform(-1, 1, (batch, m, n)).astype(np.float32)
    for cfg in [ds.KernelConfig(4, 4, 4, 8, 8), ds.KernelConfig(1, 2, 8, 16, 8)]:
        out = torch.from_numpy(c0.copy()).cuda()
        _gemm().matmul(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg,
                       out=out, alpha=0.5, beta=-1.5)
        want = gemm_f32_exact(a, b, m=m, k=k, n=n, batch=batch, stride_a=m * k,
                              stride_b=k * n, alpha=0.5, beta=-1.5, c_init=c0)
        np.testing.assert_array_equal(out.cpu().numpy().reshape(-1), want)


def test_broadcast_b_over_batch():
    ds = _dataset()
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (4, 19, 33)).astype(np.float32)
    b = rng.uniform(-1, 1, (33, 21)).astype(np.float32)
    got = _gemm().matmul(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                         ds.KernelConfig(2, 2, 2, 8, 8)).cpu().numpy()
    want = gemm_f32_exact(a, b, m=19, k=33, n=21, batch=4, stride_a=19 * 33, stride_b=0)
    np.testing.assert_array_equal(got.reshape(-1), want)


def test_unaligned_leading_dims():
    """Row pitches that are not multiples of 4 floats take the 4-byte path."""
    ds = _dataset()
    rng = np.random.default_rng(6)
    store_a = rng.uniform(-1, 1, (50, 31)).astype(np.float32)
    store_b = rng.uniform(-1, 1, (31, 23)).astype(np.float32)
    a = torch.from_numpy(store_a).cuda()[:, :27]     # lda = 31
    b = torch.from_numpy(store_b).cuda()[:27, :19]   # ldb = 23
    for cfg in [ds.KernelConfig(4, 4, 4, 8, 8), ds.KernelConfig(8, 8, 8, 16, 16)]:
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        want = gemm_f32_exact(store_a, store_b, m=50, k=27, n=19, lda=31, ldb=23).reshape(50, 19)
        np.testing.assert_array_equal(got, want)


def test_invalid_config_and_shape_errors():
    from paper_2003_06795_b200 import _native as nat
    a = torch.ones(4, 4, device="cuda")
    with pytest.raises(nat.InvalidKernelConfig):
        _gemm().matmul(a, a, (3, 4, 4, 8, 8))
    with pytest.raises(nat.BadProblemShape):
        _gemm().matmul(a, torch.ones(5, 4, device="cuda"), (4, 4, 4, 8, 8))


def test_timing_loop_positive():
    ds = _dataset()
    a = torch.rand(256, 256, device="cuda")
    ns = _gemm().time_config(a, a, ds.KernelConfig(4, 4, 4, 8, 8), reps=5)
    assert ns > 0.0
    res = _gemm().sweep_problem(a, a, ds.all_configs()[:10], reps=3)
    assert len(res) == 10 and all(v > 0 for v in res)


def test_runtime_selection_full_and_lean_library():
    """kp_gemm_auto through the compiled selector: bit-exact vs the oracle in
    the full library and in libkp_lean.so (only selector-reachable kernels),
    and both libraries choose the same config."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lean = root / "paper_2003_06795_b200" / "libkp_lean.so"
    if not lean.exists():
        pytest.skip("lean library not built")
    script = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2003_06795_b200 import gemm
from oracle.gemm_oracle import gemm_f32_exact
gemm.set_skinny(0)  # the tile selector's choice (the small-M path has its own tests)
out = []
for (m, k, n) in [(17, 27, 15), (200, 576, 64), (1, 4096, 1000), (512, 512, 512)]:
    rng = np.random.default_rng(m + k + n)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    c = gemm.matmul(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    ok = bool(np.array_equal(c, gemm_f32_exact(a, b, m=m, k=k, n=n).reshape(m, n)))
    out.append([m, k, n, list(gemm.select(m, k, n).as_tuple()), ok])
print(json.dumps(out))
'''
    res = {}
    for name, path in (("full", root / "paper_2003_06795_b200" / "libkp.so"), ("lean", lean)):
        env = dict(__import__("os").environ, KP_LIB_PATH=str(path))
        run = subprocess.run([sys.executable, "-c", script, str(root)], env=env,
                             capture_output=True, text=True, timeout=300)
        assert run.returncode == 0, run.stderr[-2000:]
        res[name] = json.loads(run.stdout.strip().splitlines()[-1])
    assert res["full"] == res["lean"]
    assert all(row[-1] for row in res["full"])


def test_pinned_pipeline_matches_device_matmul():
    """The overlapped host-buffer path (bench e2e) returns exactly what the
    device-resident call returns, also when a large problem is split into row
    blocks."""
    gemm = _gemm()
    rng = np.random.default_rng(9)
    probs, want = [], []
    # (2100, 700, 300): A is 5.9 MB -> split into row blocks (B copied once)
    for m, k, n in [(64, 64, 64), (300, 27, 70), (512, 512, 512), (2100, 700, 300)]:
        a = torch.from_numpy(rng.uniform(-1, 1, (m, k)).astype(np.float32))
        b = torch.from_numpy(rng.uniform(-1, 1, (k, n)).astype(np.float32))
        probs.append((a.pin_memory(), b.pin_memory(), torch.empty((m, n), pin_memory=True)))
        want.append(gemm.matmul(a.cuda(), b.cuda()).cpu())
    pipe = gemm.PinnedPipeline("f32")
    for _ in range(2):
        got = pipe.run(probs)
        for g, w in zip(got, want):
            assert torch.equal(g, w)


def test_pinned_pipeline_graph_replays_track_host_data():
    """graph=True captures the step once; replays read the host buffers'
    current contents (new data in the same pinned buffers -> new results)."""
    gemm = _gemm()
    rng = np.random.default_rng(10)
    shapes = [(64, 64, 64), (300, 27, 70), (2100, 700, 300)]
    probs = [(torch.empty((m, k)).pin_memory(), torch.empty((k, n)).pin_memory(),
              torch.empty((m, n), pin_memory=True)) for m, k, n in shapes]
    pipe = gemm.PinnedPipeline("f32", graph=True)
    for _ in range(3):
        for (m, k, n), (ha, hb, _) in zip(shapes, probs):
            ha.copy_(torch.from_numpy(rng.uniform(-1, 1, (m, k)).astype(np.float32)))
            hb.copy_(torch.from_numpy(rng.uniform(-1, 1, (k, n)).astype(np.float32)))
        got = pipe.run(probs)
        for (ha, hb, _), g in zip(probs, got):
            assert torch.equal(g, gemm.matmul(ha.cuda(), hb.cuda()).cpu())
    assert len(pipe._graphs) == 1


@pytest.fixture
def schedule():
    """Set the K1 tile-scheduling mode (kp_set_schedule) for one test."""
    from paper_2003_06795_b200 import _native as nat
    prev = []

    def set_mode(mode):
        prev.append(nat.lib().kp_set_schedule(mode))
    yield set_mode
    if prev:
        nat.lib().kp_set_schedule(prev[0])


@pytest.mark.parametrize("shape,ta,tb", [((70, 200, 66), False, False), ((45, 130, 97), True, True),
                                         ((64, 64, 64), False, True), ((33, 300, 40), True, False)])
def test_every_config_bit_exact_forced_stream_k(schedule, shape, ta, tb):
    """Ordered stream-K forced on small problems (grid = tiles - 1, so tiles
    are split between neighbouring CTAs): still bit-identical to the
    sequential-fmaf oracle for every config."""
    schedule(2)
    m, k, n = shape
    rng = np.random.default_rng(11)
    a_store, b_store, a, b = _operands(rng, m, k, n, ta, tb)
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta, trans_b=tb).reshape(m, n)
    bad = []
    for cfg in _dataset().all_configs():
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(cfg.as_tuple())
    assert not bad, f"{len(bad)} configs differ, first {bad[:5]}"


@pytest.mark.parametrize("mkn", [(1500, 777, 1300), (2000, 300, 2000)])
@pytest.mark.parametrize("cfg", [(1, 8, 8, 32, 8), (4, 8, 4, 16, 16), (2, 4, 4, 16, 16),
                                 (4, 8, 8, 16, 16), (1, 1, 1, 1, 64)])
def test_auto_stream_k_large_matches_one_tile_per_cta(schedule, cfg, mkn):
    """Problems with more tiles than resident CTAs take the stream-K schedule
    in auto mode (2000^2 with 64x64 tiles: two whole waves, then stream-K over
    the rest); C must equal the one-tile-per-CTA result bit for bit and the
    oracle on sampled rows."""
    gemm = _gemm()
    m, k, n = mkn
    rng = np.random.default_rng(12)
    a_store, b_store, a, b = _operands(rng, m, k, n, False, False)
    schedule(1)
    got = gemm.matmul(a, b, cfg).cpu().numpy()
    schedule(0)
    classic = gemm.matmul(a, b, cfg).cpu().numpy()
    np.testing.assert_array_equal(got, classic)
    rows = np.array([0, 1, 255, 256, 700, 1023, 1024, 1499, m - 1])
    want = gemm_f32_exact(np.ascontiguousarray(a_store[rows]), b_store, m=len(rows), k=k,
                          n=n).reshape(len(rows), n)
    np.testing.assert_array_equal(got[rows], want)


def test_stream_k_batched_and_back_to_back(schedule):
    """Stream-K over a strided batch (units span batch entries) and many
    back-to-back launches (flag ring reuse) stay exact."""
    schedule(2)
    ds = _dataset()
    rng = np.random.default_rng(13)
    batch, m, k, n = 5, 96, 160, 80
    a = rng.uniform(-1, 1, (batch, m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (batch, k, n)).astype(np.float32)
    want = gemm_f32_exact(a, b, m=m, k=k, n=n, batch=batch, stride_a=m * k, stride_b=k * n)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for cfg in [ds.KernelConfig(4, 4, 4, 8, 8), ds.KernelConfig(2, 2, 8, 16, 8)]:
        outs = [_gemm().matmul(ta, tb, cfg) for _ in range(300)]
        for o in outs[::37] + outs[-1:]:
            np.testing.assert_array_equal(o.cpu().numpy().reshape(-1), want)


def test_stream_k_needs_beta_zero(schedule):
    """beta != 0 keeps the one-tile-per-CTA schedule (C is read), still exact."""
    schedule(2)
    ds = _dataset()
    rng = np.random.default_rng(14)
    m, k, n = 70, 90, 60
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    c0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    out = torch.from_numpy(c0.copy()).cuda()
    _gemm().matmul(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                   ds.KernelConfig(2, 2, 2, 8, 8), out=out, alpha=2.0, beta=0.5)
    want = gemm_f32_exact(a, b, m=m, k=k, n=n, alpha=2.0, beta=0.5, c_init=c0)
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1), want)


@pytest.mark.parametrize("ta", [False, True])
def test_every_config_bit_exact_tall_b_transposed(ta):
    """m >= 2048 with B transposed stages B transposed into the chunk layout
    (copy_transpose, FFMA2 column pairs); ragged m/n/k edges included."""
    m, k, n = 2053, 45, 37
    rng = np.random.default_rng(15)
    a_store, b_store, a, b = _operands(rng, m, k, n, ta, True)
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta, trans_b=True).reshape(m, n)
    bad = []
    for cfg in _dataset().all_configs():
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(cfg.as_tuple())
    assert not bad, f"{len(bad)} configs differ, first {bad[:5]}"


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_runtime_selection_every_layout(ta, tb):
    """kp_gemm_auto has a compiled selector for every FP32 operand layout
    (the sweep + prune + decision-tree pipeline ran per layout) and the
    selected kernel is bit-exact vs the oracle."""
    gemm = _gemm()
    for (m, k, n) in [(17, 27, 15), (200, 576, 64), (2100, 64, 96)]:
        rng = np.random.default_rng(m + 3 * k + 7 * n)
        a_store, b_store, a, b = _operands(rng, m, k, n, ta, tb)
        cfg = gemm.select(m, k, n, trans_a=ta, trans_b=tb)
        got = gemm.matmul(a, b).cpu().numpy()
        want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta,
                              trans_b=tb).reshape(m, n)
        np.testing.assert_array_equal(got, want, err_msg=f"{(m, k, n)} {cfg}")


def test_registered_torch_op():
    """torch.ops.kernelprune.matmul is the runtime-selected library call."""
    gemm = _gemm()
    op = gemm.torch_op()
    a = torch.rand(300, 200, device="cuda")
    b = torch.rand(200, 100, device="cuda")
    got = op(a, b, "f32")
    assert torch.equal(got, gemm.matmul(a, b))
    # the fake implementation propagates shapes without launching
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        fa, fb = torch.empty(7, 5, device="cuda"), torch.empty(5, 3, device="cuda")
        assert op(fa, fb, "f32").shape == (7, 3)


def test_batched_runtime_selection():
    """Strided-batched problems dispatch through the batched selector
    (select_f32_nn_b8, kp_select_ex with batch > 1) and stay bit-exact."""
    import ctypes
    from paper_2003_06795_b200 import _native as nat
    gemm = _gemm()
    for (bt, m, k, n) in [(8, 784, 576, 64), (3, 196, 2304, 256), (8, 49, 512, 2048)]:
        rng = np.random.default_rng(bt * m + k)
        a = rng.uniform(-1, 1, (bt, m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (bt, k, n)).astype(np.float32)
        cfg = gemm.select(m, k, n, batch=bt)
        assert gemm.auto_config(m, k, n, batch=bt) == cfg
        got = gemm.matmul(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        want = gemm_f32_exact(a, b, m=m, k=k, n=n, batch=bt, stride_a=m * k, stride_b=k * n,
                              stride_c=m * n).reshape(bt, m, n)
        np.testing.assert_array_equal(got, want, err_msg=f"{(bt, m, k, n)} {cfg}")
        # kp_gemm_auto reports the batched tree's pick
        d, da, db, dc = gemm.describe(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
        chosen = nat.KpConfig()
        nat.check(nat.lib().kp_gemm_auto(nat.F32_SIMT, ctypes.byref(d), da.data_ptr(),
                                         db.data_ptr(), dc.data_ptr(), None, ctypes.byref(chosen)))
        torch.cuda.synchronize()
        assert chosen.as_tuple() == cfg.as_tuple()


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("shape", [(320, 96, 192), (256, 100, 160)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_every_config_bit_exact_aligned_interior(schedule, ta, tb, shape, mode):
    """16-byte aligned operands with whole interior tiles and several K
    slices: the hoisted interior copy plan (CopyPlan, thread tiles <= 32
    outputs) and the per-slice interior copies (8x8 tiles) run, including
    from a mid-tile k-slice (forced stream-K, mode 2) and before a ragged
    last slice (k = 100); every config bit-identical to the oracle."""
    schedule(mode)
    m, k, n = shape
    rng = np.random.default_rng(21)
    a_store, b_store, a, b = _operands(rng, m, k, n, ta, tb)
    want = gemm_f32_exact(a_store, b_store, m=m, k=k, n=n, trans_a=ta, trans_b=tb).reshape(m, n)
    bad = []
    for cfg in _dataset().all_configs():
        got = _gemm().matmul(a, b, cfg).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(cfg.as_tuple())
    assert not bad, f"{len(bad)} configs differ, first {bad[:5]}"
