"""GPU-vs-oracle parity of libsagips on one B200 (through the C ABI).

Tolerances (from BASELINE.json north_star): bit-exact
RNG counters, bootstrap indices, histogram counts and reference / shard
rows; 1e-5 relative for fp32 events and losses; 1e-3 relative (with the R24
floor) for fp32 gradients; parameters after one Adam step within 2 lr."""
import numpy as np
import pytest

from oracle import exchange as xc
from oracle import gan, mlp, proxy
from oracle import philox as px
from tests import inputs, kink
from tests.gpu_util import assert_grad_close, assert_rel, flat, lib, oracle_config, sync_params, unflat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _stream():
    import ctypes
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_ctx(cfg):
    from paper_2407_00051_b200 import runtime
    return runtime.make_context(cfg)


# ---------------------------------------------------------------- sampler
@pytest.mark.parametrize("k,m,bins", [(1, 1, 64), (3, 5, 64), (64, 16, 64), (7, 1023, 64), (1024, 1024, 64),
                                       (64, 16, 1), (7, 1023, 200), (1024, 1024, 200), (1024, 1024, 0)])
def test_sample_events_parity(k, m, bins):
    """bins 200: the shared histograms no longer fit the lane-column layout
    (one copy per block instead); bins 0: no histogram (hist = NULL)."""
    L = lib()
    seed, step, rank = 0xC0FFEE12345678, 123457, 3
    c32 = inputs.coefficients(k * 31 + m, k).astype(np.float32)
    c_t = torch.tensor(c32, device="cuda")
    ev = torch.empty(k * m * 2, dtype=torch.float32, device="cuda")
    hist = torch.zeros(2 * (max(bins, 1) + 2), dtype=torch.int32, device="cuda")
    L.sample_events(c_t.data_ptr(), k, m, seed, step, rank, px.STREAM_FAKE, ev.data_ptr(),
                    hist.data_ptr() if bins else 0, bins, (0.0, 0.0), (4.0, 4.0), _stream())
    torch.cuda.synchronize()
    y_gpu = ev.cpu().numpy().reshape(-1, 2)
    u = proxy.fake_uniforms(seed, step, rank, k * m)
    y32 = proxy.sample_events_f32(c32, m, u)
    assert np.array_equal(y_gpu, y32)                       # same fp32 operations -> bit-exact
    assert_rel(y_gpu, proxy.sample_events(c32.astype(np.float64), m, u), 1e-5, 1e-6, "events vs fp64")
    if not bins:
        return
    h = hist.cpu().numpy().astype(np.int64).reshape(2, bins + 2)
    for o in range(2):
        assert np.array_equal(h[o], proxy.histogram_f32(y32[:, o], 0.0, 4.0, bins))


def test_sample_events_rejects_bad_args():
    L = lib()
    with pytest.raises(L.SagipsError):
        L.sample_events(None, 1, 1, 0, 0, 0, 5, None)


# ---------------------------------------------------------------- init
@pytest.mark.parametrize("preset,kw", [(0, {}), (1, dict(param_samples=16, events_per_sample=61))])
def test_create_matches_oracle_init(preset, kw):
    L = lib()
    cfg = L.config_init(preset, rank=0, **kw)
    cfg.reference_rows = 2 * cfg.param_samples * cfg.events_per_sample + 7   # ragged
    cfg.shard_rows = cfg.param_samples * cfg.events_per_sample + 3
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    ref32 = proxy.make_reference_f32(ocfg.seed, ocfg.true_params, ocfg.reference_rows)
    assert np.array_equal(ctx.get(L.T_REFERENCE).reshape(-1, 2), ref32)
    assert np.array_equal(ctx.get(L.T_SHARD).reshape(-1, 2), st.shard32)
    for which, ws in ((L.T_GEN_W, st.gW), (L.T_DISC_W, st.dW)):
        assert_rel(ctx.get(which), flat(ws), 2e-5, 2e-6, "kaiming init")
    assert np.all(ctx.get(L.T_GEN_B) == 0) and np.all(ctx.get(L.T_DISC_B) == 0)


# ---------------------------------------------------------------- one step
def _check_step(cfg, t=0, disc_band=kink.BAND_FP32, fake_dev=0.0, g_outliers=0.0):
    L = lib()
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, cfg.rank)
    sync_params(ctx, st)
    d_before = flat(st.dW).copy()
    d_params0 = ([w.copy() for w in st.dW], [b.copy() for b in st.db])
    g_params0 = ([w.copy() for w in st.gW], [b.copy() for b in st.gb])
    ctx.train_step(t, L.STEP_LOCAL_ONLY, _stream())
    out = gan.local_step(ocfg, st, t)
    # the G step is checked against the oracle's G step through the GPU's own
    # updated discriminator: Adam's first step is +-lr for any |g| >> eps, so a
    # sign flip of a near-zero D gradient legitimately moves that weight by 2 lr
    gpu_d = (unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db))
    _, g_cache = mlp.forward(g_params0[0], g_params0[1], out["z"], ocfg.leaky_slope)
    og = gan.generator_step(ocfg, gpu_d[0], gpu_d[1], g_params0[0], g_cache, out["raw"], out["u"], out["y"])
    kd = kink.step_deviation(ocfg, d_params0, gpu_d, g_params0, out, disc_band, fake_dev)
    N = ocfg.n_events
    stats = ctx.get(L.T_STATS)
    assert stats.nonfinite == 0
    assert_rel(ctx.get(L.T_NOISE), out["z"].reshape(-1), 1e-5, 1e-6, "noise")
    assert_rel(ctx.get(L.T_RAW), out["raw"].reshape(-1), 1e-5, 1e-5, "raw")
    assert np.array_equal(ctx.get(L.T_REAL_IDX), out["real_idx"].astype(np.uint32))   # bootstrap indices
    ev = ctx.get(L.T_EVENTS).reshape(-1, 2)
    assert np.array_equal(ev[:N], st.shard32[out["real_idx"]])                           # real rows exact
    assert_rel(ev[N:], out["y"], 1e-5, 1e-5, "fake events")
    hist = ctx.get(L.T_HIST).astype(np.int64).reshape(2, 2, -1)
    assert np.array_equal(hist[0], out["hist"][0])                                       # real hist exact
    assert np.abs(hist[1] - out["hist"][1]).sum() <= max(4, N // 20000)                   # R22: ULP edges
    assert_rel(ctx.get(L.T_LOGITS_D), out["logits_d"], 1e-4, 1e-4, "D logits")
    assert stats.loss_d == pytest.approx(out["loss_d"], rel=1e-5)
    assert_grad_close(ctx.get(L.T_DISC_DW), flat(out["dW_d"]), 1e-3, "dW_D", kd["dW_d"])
    assert_grad_close(ctx.get(L.T_DISC_DB), flat(out["db_d"]), 1e-3, "db_D", kd["db_d"])
    # one Adam step moves each parameter by at most ~lr; allow 2 lr
    assert np.max(np.abs(ctx.get(L.T_DISC_W) - flat(st.dW))) <= 2.0 * ocfg.disc_lr + 1e-6
    assert np.max(np.abs(ctx.get(L.T_DISC_W) - d_before)) > 0
    assert stats.loss_g == pytest.approx(og["loss_g"], rel=1e-5)
    # against the independent trajectory: its D differs from the GPU's by up to
    # 2 lr where an Adam step saw a near-zero gradient of the other sign (above),
    # which moves L_G by up to ~1e-5 relative at these sizes; 1e-5 holds through
    # the GPU's D (above) and, independent, at full size (test_full_size_...)
    assert stats.loss_g == pytest.approx(out["loss_g"], rel=1e-4)
    assert_rel(ctx.get(L.T_LOGITS_G), og["logits_g"], 1e-4, 1e-4, "G logits")
    nout = lambda v: int(np.ceil(g_outliers * np.size(v))) if g_outliers else 0  # noqa: E731
    assert_grad_close(ctx.get(L.T_DY), og["dy"], 1e-3, "dy", kd["dy"], nout(og["dy"]))
    assert_grad_close(ctx.get(L.T_DRAW), og["draw"], 1e-3, "draw", kd["draw"], nout(og["draw"]))
    assert_grad_close(ctx.get(L.T_GEN_DW), og["packet"], 1e-3, "packet dW_G", kd["packet"], nout(og["packet"]))
    assert_grad_close(ctx.get(L.T_GEN_DB), flat(og["db_g"]), 1e-3, "db_G", kd["db_g"], nout(flat(og["db_g"])))
    return ctx, st, out


def test_step_many_histogram_bins():
    """hist_bins = 300: the step's four shared histograms exceed the
    lane-column layout (one copy per block); paper widths, fused kernels."""
    L = lib()
    _check_step(L.config_init(1, seed=8, param_samples=64, events_per_sample=64, hist_bins=300), t=1,
                disc_band=kink.BAND_BF16X3, g_outliers=1e-3)  # R27 mixed-pattern flips, as the k = 63 case


def test_step_desk():
    _check_step(lib().config_init(0, seed=5))


@pytest.mark.parametrize("preset,k,m,G", [(0, 16, 37, 65), (1, 64, 61, 257)])
def test_step_tabulated_sampler(preset, k, m, G):
    """The whole step with the tabulated-CDF sampler:
    reference data, fake rows, fake histogram and the sampler backward from
    the tabulated density; everything else as the quadratic step.  Paper
    widths at the ragged test's 2N = 7,808 rows: the bf16x2 wgrad (R28)
    averages its hi-plane rounding over the rows."""
    L = lib()
    cfg = L.config_init(preset, seed=13, param_samples=k, events_per_sample=m, reference_rows=2 * k * m + 5,
                        shard_rows=k * m + 3, sampler=L.SAMPLER_TABULATED, sampler_grid=G)
    for j, v in enumerate((0.3, 2.0, 1.2, 0.7, 1.5, 3.0)):   # (w, b, c) per observable
        cfg.true_params[j] = v
    cfg.hist_lo[0] = cfg.hist_lo[1] = 0.0
    cfg.hist_hi[0] = cfg.hist_hi[1] = 1.0
    # the fake events agree to the asserted 1e-5 + 1e-5 |y| <= 2e-5 (y in [0, 1]): that input
    # deviation widens the kink band (tests/kink.py), and up to 0.1% of the G-step gradient
    # elements may carry a mixed-pattern kink flip (assert_grad_close outliers)
    ctx, st, out = _check_step(cfg, t=2, disc_band=kink.BAND_BF16X3 if preset == 1 else kink.BAND_FP32,
                               fake_dev=2e-5, g_outliers=1e-3)
    # the constrained output holds (w, b, c) per observable
    assert_rel(ctx.get(L.T_C), out["c"].reshape(-1), 1e-5, 1e-6, "constrained (w, b, c)")


@pytest.fixture
def fused_env(request, monkeypatch):
    """SAGIPS_FUSED: "1" the fused discriminator kernels (k_dfwd, k_gstep;
    default), "0" the per-layer tcgen05 kernels; "1p": fused, with the G_4
    planes written by k_dfwd instead of regenerated from dz + sign bits by
    the next pass (SAGIPS_GEN_G=0)."""
    monkeypatch.setenv("SAGIPS_FUSED", request.param[0])
    monkeypatch.setenv("SAGIPS_GEN_G", "0" if request.param == "1p" else "1")
    return request.param


@pytest.mark.parametrize("impl,fused_env,k", [(0, "1", 64), (0, "1p", 64), (0, "0", 64), (1, "1", 64),
                                               (0, "1", 63), (0, "0", 63)], indirect=["fused_env"])
def test_step_paper_widths_ragged(impl, fused_env, k):
    """paper widths, 2N = 7,808 rows (ragged 128-row tiles), step 3, rank 1;
    impl 0 = tcgen05 bf16x3 hidden layers (fused kernels or per-layer
    kernels), 1 = CUDA-core fp32.  k = 63: N = 3,843 is odd, so the fake
    rows (X + 2N floats) are only 8-byte aligned; there two dy elements sit
    3% past the kink band with identical values from the fused and the
    per-layer kernels (a LeakyReLU decision, R27), so up to 0.1% of the
    G-step elements may be kink outliers bounded by max|ref|."""
    L = lib()
    _check_step(L.config_init(1, seed=9, param_samples=k, events_per_sample=61, world=2, rank=1, group_size=2,
                              disc_impl=impl), t=3, disc_band=kink.BAND_BF16X3 if impl == 0 else kink.BAND_FP32,
                g_outliers=1e-3 if k == 63 else 0.0)


@pytest.mark.parametrize("k,m", [(1, 1), (3, 5), (2, 64), (1, 129)])
def test_step_paper_widths_tiny(k, m):
    """paper widths (fused kernels, fp32-class) at degenerate sizes: one
    event, one partial 128-row tile (2N = 2, 30, 256, 258 rows; a single CTA
    slot has all the work, the other none).  Sums over so few rows do not
    average the wgrad's bf16 rounding of H (R28, 2^-9 per product) below the
    1e-3 bar of the large tests, so every element is held to the first-order
    bound of the split scheme instead (tests/bf16_bound.py, scheme 'split')."""
    from tests import bf16_bound
    L = lib()
    cfg = L.config_init(1, seed=13, param_samples=k, events_per_sample=m)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    d0 = ([w.copy() for w in st.dW], [b.copy() for b in st.db])
    g0 = ([w.copy() for w in st.gW], [b.copy() for b in st.gb])
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    out = gan.local_step(ocfg, st, 0)
    ev = ctx.get(L.T_EVENTS).reshape(-1, 2)
    N = k * m
    assert_rel(ev[N:], out["y"], 1e-5, 1e-5, "fake events")
    gpu_d = (unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db))
    _, g_cache = mlp.forward(g0[0], g0[1], out["z"], ocfg.leaky_slope)
    og = gan.generator_step(ocfg, gpu_d[0], gpu_d[1], g0[0], g_cache, out["raw"], out["u"], out["y"])
    bf16_bound.use_scheme("split")
    try:
        tol = bf16_bound.step_tolerances(ocfg, d0, gpu_d, g0, out)
    finally:
        bf16_bound.use_scheme("bf16")
    s = ctx.get(L.T_STATS)
    assert abs(s.loss_d - out["loss_d"]) <= 2 * tol["loss_d"] + 1e-5 * abs(out["loss_d"]), (s.loss_d, out["loss_d"])
    assert abs(s.loss_g - og["loss_g"]) <= 2 * tol["loss_g"] + 1e-5 * abs(og["loss_g"]), (s.loss_g, og["loss_g"])
    for name, which, ref in (("dW_d", L.T_DISC_DW, flat(out["dW_d"])), ("db_d", L.T_DISC_DB, flat(out["db_d"])),
                             ("dy", L.T_DY, og["dy"]), ("draw", L.T_DRAW, og["draw"]),
                             ("packet", L.T_GEN_DW, og["packet"]), ("db_g", L.T_GEN_DB, flat(og["db_g"]))):
        g = ctx.get(which).astype(np.float64)
        r = np.asarray(ref, dtype=np.float64).reshape(-1)
        allowed = tol[name] + 1e-5 * np.abs(r) + 1e-6 * np.max(np.abs(r))  # + fp32 rounding of the rest
        ratio = np.abs(g - r) / allowed
        assert np.all(ratio <= 1.0), f"{name}: {int(np.sum(ratio > 1))} elements outside the split bound (worst {ratio.max():.3g})"


@pytest.mark.parametrize("fused_env,k,m", [("1", 128, 1024), ("1p", 128, 1024), ("0", 128, 1024), ("1", 125, 1021),
                                           ("0", 125, 1021)],
                         indirect=["fused_env"])
def test_bf16_step_elementwise(fused_env, k, m):
    """SAGIPS_PREC_BF16 (C5's precision): discriminator GEMMs in bf16 with fp32
    accumulation, at 2N = 2^18 rows.  Every element of dW_D, db_D, dy, draw,
    the packet and db_G, and both losses, within the first-order bf16 error
    bound of the oracle's own values (tests/bf16_bound.py: operand rounding
    2^-9 propagated through |h| |W| forward and backward, x2) plus the
    LeakyReLU kink deviation with per-element bands and a 1e-4 max|ref|
    floor.  The G step is compared through the GPU's updated D (as the fp32
    step tests).  k = 125, m = 1021: N = 127,625 and 2N = 255,250 rows, ragged
    last 128-row tiles through the fused kernels and the G_4 regeneration."""
    from tests import bf16_bound
    L = lib()
    cfg = L.config_init(1, seed=4, param_samples=k, events_per_sample=m, precision=L.PREC_BF16)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    d0 = ([w.copy() for w in st.dW], [b.copy() for b in st.db])
    g0 = ([w.copy() for w in st.gW], [b.copy() for b in st.gb])
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    out = gan.local_step(ocfg, st, 0)
    gpu_d = (unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db))
    _, g_cache = mlp.forward(g0[0], g0[1], out["z"], ocfg.leaky_slope)
    og = gan.generator_step(ocfg, gpu_d[0], gpu_d[1], g0[0], g_cache, out["raw"], out["u"], out["y"])
    tol = bf16_bound.step_tolerances(ocfg, d0, gpu_d, g0, out)
    s = ctx.get(L.T_STATS)
    assert abs(s.loss_d - out["loss_d"]) <= 2 * tol["loss_d"] + 1e-6, (s.loss_d, out["loss_d"], tol["loss_d"])
    assert abs(s.loss_g - og["loss_g"]) <= 2 * tol["loss_g"] + 1e-6, (s.loss_g, og["loss_g"], tol["loss_g"])
    worst = {}
    for name, which, ref in (("dW_d", L.T_DISC_DW, flat(out["dW_d"])), ("db_d", L.T_DISC_DB, flat(out["db_d"])),
                             ("dy", L.T_DY, og["dy"]), ("draw", L.T_DRAW, og["draw"]),
                             ("packet", L.T_GEN_DW, og["packet"]), ("db_g", L.T_GEN_DB, flat(og["db_g"]))):
        g = ctx.get(which).astype(np.float64)
        r = np.asarray(ref, dtype=np.float64).reshape(-1)
        allowed = tol[name] + 1e-4 * np.max(np.abs(r))
        ratio = np.abs(g - r) / allowed
        worst[name] = float(ratio.max())
        assert np.all(ratio <= 1.0), f"{name}: {int(np.sum(ratio > 1))} elements outside the bf16 bound (worst {ratio.max():.3g})"
    print("bf16 step: worst error / bound", worst)


def test_full_step_applies_generator_update():
    L = lib()
    cfg = L.config_init(0, seed=11)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    ctx.train_step(0, 0, _stream())
    out = gan.local_step(ocfg, st, 0)
    gan.apply_generator(ocfg, st, out["packet"], out["db_g"])
    assert_grad_close(ctx.get(L.T_REDUCED), out["packet"], 1e-3, "reduced (mode NONE)")
    assert np.max(np.abs(ctx.get(L.T_GEN_W) - flat(st.gW))) <= 2.0 * ocfg.gen_lr + 1e-7
    assert np.max(np.abs(ctx.get(L.T_GEN_B) - flat(st.gb))) <= 2.0 * ocfg.gen_lr + 1e-7


def test_loss_curves_200_steps_desk():
    """C1: 200 steps; 10-step moving averages of L_D and L_G within 2% (R25)."""
    L = lib()
    cfg = L.config_init(0, seed=3)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    gl, ol = [], []
    for t in range(200):
        ctx.train_step(t, 0, _stream())
        s = ctx.get(L.T_STATS)
        gl.append((s.loss_d, s.loss_g))
        o = gan.local_step(ocfg, st, t)
        gan.apply_generator(ocfg, st, o["packet"], o["db_g"])
        ol.append((o["loss_d"], o["loss_g"]))
    g = np.array(gl)
    o = np.array(ol)
    kern = np.ones(10) / 10
    for j in range(2):
        gm = np.convolve(g[:, j], kern, mode="valid")
        om = np.convolve(o[:, j], kern, mode="valid")
        assert np.max(np.abs(gm - om) / np.abs(om)) < 0.02


def test_step_order_and_exchange_state_errors():
    L = lib()
    ctx = make_ctx(L.config_init(0))
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    with pytest.raises(L.SagipsError) as e:
        ctx.pull_generator_grad(0, _stream())
    assert e.value.status == 6
    ctx.push_generator_grad(0, _stream())
    ctx.pull_generator_grad(0, _stream())
    with pytest.raises(L.SagipsError) as e:
        ctx.train_step(0, 0, _stream())
    assert e.value.status == 6


def test_full_size_paper_step_sampled():
    """C2 at full size (k = m = 1024, 2N = 2^21 rows) in the launch
    configuration bench.py times (fused discriminator kernels): both losses
    (1e-5), the histograms, sampled events / indices and every gradient
    against the independent oracle."""
    L = lib()
    cfg = L.config_init(1, seed=2)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    g0 = ([w.copy() for w in st.gW], [b.copy() for b in st.gb])
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    out = gan.local_step(ocfg, st, 0)
    N = ocfg.n_events
    s = ctx.get(L.T_STATS)
    assert s.loss_d == pytest.approx(out["loss_d"], rel=1e-5)
    assert s.loss_g == pytest.approx(out["loss_g"], rel=1e-5)
    idx = inputs.sample_indices(1, N, 4096)
    ev = ctx.get(L.T_EVENTS).reshape(-1, 2)
    assert np.array_equal(ctx.get(L.T_REAL_IDX)[idx], out["real_idx"][idx].astype(np.uint32))
    assert_rel(ev[N + idx], out["y"][idx], 1e-5, 1e-5, "fake events (sampled)")
    hist = ctx.get(L.T_HIST).astype(np.int64).reshape(2, 2, -1)
    assert np.array_equal(hist[0], out["hist"][0])
    assert np.abs(hist[1] - out["hist"][1]).sum() <= max(4, N // 20000)  # R22: fake events within an ULP of an edge
    # every gradient of the step against the independent oracle (its own D
    # step and Adam, then its own G step), sampled rows for dy.  The G-step
    # quantities per sample (draw) and per row (dy) are checked at 1e-3
    # through the GPU's updated D and against the independent trajectory at
    # 1e-2 (draw elementwise -- both on dy's tolerance carried through the
    # sum over events, see below --, dy in relative L2 norm: single rows can cancel):
    # after one Adam step a near-zero D gradient of the other sign moves that
    # weight by 2 lr, which they are sensitive to (the sums over samples, the
    # packet and db_G, hold 1e-3 either way)
    assert_grad_close(ctx.get(L.T_GEN_DW), out["packet"], 1e-3, "packet dW_G")
    assert_grad_close(ctx.get(L.T_GEN_DB), flat(out["db_g"]), 1e-3, "db_G")
    assert_grad_close(ctx.get(L.T_DISC_DW), flat(out["dW_d"]), 1e-3, "dW_D")
    assert_grad_close(ctx.get(L.T_DISC_DB), flat(out["db_d"]), 1e-3, "db_D")
    # draw_s = sum over the sample's 1024 events of dy u^j softplus': it
    # cancels heavily, so its tolerance is dy's (1e-3 with the R24 floor)
    # carried through that linear map on magnitudes: sum tol(dy) |u^j| softplus'
    m = ocfg.events_per_sample
    tol_dy = 1e-3 * np.maximum(np.abs(out["dy"]), 1e-2 * np.max(np.abs(out["dy"])))
    _, draw_mag = proxy.sampler_backward(tol_dy, out["u"], out["raw"], m)
    tol_draw = (1e-3 * np.abs(out["draw"]) + draw_mag).reshape(-1)
    # (no kink band at this size -- R27's forced-branch deviation over 2^21
    # rows is not computed -- so up to 0.1% of the samples may hold a row whose
    # LeakyReLU' decision differs: each within 10x the tolerance)
    def check_draw(ref, scale, what):
        err = np.abs(ctx.get(L.T_DRAW).astype(np.float64) - np.asarray(ref).reshape(-1))
        ratio = err / (scale * tol_draw)
        bad = np.flatnonzero(ratio > 1)
        assert bad.size <= ratio.size // 1000 and ratio.max() <= 10, \
            f"{what}: {bad.size} of {ratio.size} outside (worst {ratio.max():.3g} at {bad[:6]})"
    check_draw(out["draw"], 10.0, "draw (independent)")
    dyg, dyo = ctx.get(L.T_DY).reshape(-1, 2).astype(np.float64), out["dy"]
    assert np.linalg.norm(dyg - dyo) <= 1e-2 * np.linalg.norm(dyo), "dy (independent, relative L2)"
    gpu_d = (unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db))
    _, g_cache = mlp.forward(g0[0], g0[1], out["z"], ocfg.leaky_slope)
    og = gan.generator_step(ocfg, gpu_d[0], gpu_d[1], g0[0], g_cache, out["raw"], out["u"], out["y"])
    assert s.loss_g == pytest.approx(og["loss_g"], rel=1e-5)
    check_draw(og["draw"], 1.0, "draw (through the GPU's D)")
    # R27 at full size: no kink band is computed over 2^20 rows x 512
    # LeakyReLU decisions, so up to 0.25% of the sampled elements may carry a
    # flipped decision (observed on B200: 3 of 4,096 rows), each within max|ref|
    assert_grad_close(ctx.get(L.T_DY).reshape(-1, 2)[idx], og["dy"][idx], 1e-3, "dy (through the GPU's D, sampled)",
                      outliers=idx.size * 2 // 400)


def test_max_size_fp32_step_sampled_rows():
    """The largest configuration (C5's size: k = 1,024, m = 16,384, N = 2^24,
    2N = 2^25 rows) through the fp32-class fused kernels, checked row by row
    where the oracle can compute one row alone (the full oracle step does not
    fit here): the generator's c; for 4,096 sampled events (incl. the first,
    the last and sample boundaries) the bootstrap index, the real row and
    the fake event (bit-exact / 1e-5), the D logits of both rows from the
    GPU's own rows and the pre-step D, and the G step's logit and dy through
    the GPU's updated D (1e-4 / 1e-3 with the R24 floor and R27 outliers)."""
    L = lib()
    k, m = 1024, 16384
    N = k * m
    cfg = L.config_init(1, seed=6, param_samples=k, events_per_sample=m, reference_rows=2 * N, shard_rows=N)
    ctx = make_ctx(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(oracle_config(L.config_init(1, seed=6)), 0)  # same seed and model: same initial weights
    sync_params(ctx, st)
    d0 = ([w.copy() for w in st.dW], [b.copy() for b in st.db])
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    a = ocfg.leaky_slope
    raw, _ = mlp.forward(st.gW, st.gb, gan.noise(ocfg, 0, 0), a)
    c = proxy.constrain(raw).reshape(k, 2, 3)
    assert_rel(ctx.get(L.T_C).reshape(k, 2, 3), c, 1e-5, 1e-6, "constrained parameters c")
    idx = np.unique(np.concatenate([[0, 1, m - 1, m, N // 2, N - 2, N - 1], inputs.sample_indices(6, N, 4096)]))
    seed = ocfg.seed
    u = np.stack([px.uniform_open01(px.words(seed, px.STREAM_FAKE, 0, 0, 2 * int(e), 2)) for e in idx])
    s_of = idx // m
    y = np.stack([proxy.quantile(u[:, o], c[s_of, o, 0], c[s_of, o, 1], c[s_of, o, 2]) for o in range(2)], axis=1)
    ridx = np.array([proxy.lemire_index(px.words(seed, px.STREAM_REAL, 0, 0, int(e), 1), N)[0] for e in idx])
    sidx = np.array([proxy.lemire_index(px.words(seed, px.STREAM_SHARD, 0, 0, int(j), 1), 2 * N)[0] for j in ridx])
    uref = np.stack([px.uniform_open01(px.words(seed, px.STREAM_REF, 0, 0, 2 * int(r), 2)) for r in sidx])
    x32 = proxy.sample_events_f32(np.repeat(np.asarray(ocfg.true_params, dtype=np.float32).reshape(1, 6), idx.size, axis=0),
                                  1, uref)
    ev = ctx.get(L.T_EVENTS).reshape(-1, 2)
    assert np.array_equal(ctx.get(L.T_REAL_IDX)[idx], ridx.astype(np.uint32)), "bootstrap indices"
    assert np.array_equal(ev[idx], x32), "real rows"
    assert_rel(ev[N + idx], y, 1e-5, 1e-5, "fake events")
    # the D step's logits of the sampled real and fake rows (the GPU's rows, the pre-step D)
    rows = np.concatenate([idx, N + idx])
    zD, _ = mlp.forward(d0[0], d0[1], ev[rows].astype(np.float64), a)

    def logits_close(gpu, ref, what):  # 1e-4; up to 0.1% of the rows within 10x (a LeakyReLU decision, R27)
        ratio = np.abs(np.asarray(gpu, dtype=np.float64) - ref) / (1e-4 + 1e-4 * np.abs(ref))
        bad = np.flatnonzero(ratio > 1)
        assert bad.size <= ratio.size // 1000 and ratio.max() <= 10, f"{what}: {bad.size} rows, worst {ratio.max():.3g}"
    logits_close(ctx.get(L.T_LOGITS_D)[rows], zD[:, 0], "D logits (sampled rows)")
    # the G step through the GPU's updated D: logit and dy of each sampled fake row
    gpu_d = (unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db))
    zG, cache = mlp.forward(gpu_d[0], gpu_d[1], ev[N + idx].astype(np.float64), a)
    logits_close(ctx.get(L.T_LOGITS_G)[idx], zG[:, 0], "G logits (sampled rows)")
    dzG = (mlp.sigmoid(zG[:, 0]) - 1.0) / N
    _, _, dy = mlp.backward(gpu_d[0], cache, dzG[:, None], a)
    assert_grad_close(ctx.get(L.T_DY).reshape(-1, 2)[idx], dy, 1e-3, "dy (sampled rows)",
                      outliers=idx.size * 2 // 400)
    # the sampler backward of whole samples (first, middle, last) from the
    # GPU's own dy: the oracle's sums over the sample's 16,384 events in fp64;
    # the GPU's fp32 reduction within 1e-5 of the sum of magnitudes
    dy_all = ctx.get(L.T_DY).reshape(-1, 2).astype(np.float64)
    draw_gpu = ctx.get(L.T_DRAW).reshape(k, 6).astype(np.float64)
    for smp in (0, k // 2, k - 1):
        e0 = smp * m
        us = px.uniform_open01(px.words(seed, px.STREAM_FAKE, 0, 0, 2 * e0, 2 * m)).reshape(m, 2)
        dys = dy_all[e0:e0 + m]
        _, draw_s = proxy.sampler_backward(dys, us, raw[smp][None, :], m)
        _, mag = proxy.sampler_backward(np.abs(dys), us, raw[smp][None, :], m)
        assert np.all(np.abs(draw_gpu[smp] - draw_s[0]) <= 1e-5 * mag[0] + 1e-30), (smp, draw_gpu[smp], draw_s[0])


def test_step_is_deterministic():
    """Two contexts from the same state produce bit-identical losses,
    gradients, events and parameters (fixed-order reductions everywhere; the
    dynamic tile schedule only moves tiles whose outputs do not depend on the
    CTA).  Paper widths, 2N = 2^18 rows (several tiles per CTA)."""
    L = lib()
    outs = []
    for _ in range(2):
        cfg = L.config_init(1, seed=13, param_samples=128, events_per_sample=1024)
        ctx = make_ctx(cfg)
        for t in range(2):
            ctx.train_step(t, L.STEP_LOCAL_ONLY, _stream())
        torch.cuda.synchronize()
        outs.append({w: ctx.get(w) for w in (L.T_DISC_DW, L.T_DISC_DB, L.T_DISC_W, L.T_DY, L.T_GEN_DW, L.T_LOGITS_D,
                                              L.T_EVENTS)})
        s = ctx.get(L.T_STATS)
        outs[-1]["loss"] = np.array([s.loss_d, s.loss_g])
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_kernel_times_cover_the_layer_passes():
    """sagips_kernel_times: the tcgen05 discriminator kernels of a paper-width
    step are all timed (positive): the D step's per-layer passes (or the fused
    D forward) and the G step's passes (or the fused G step); their sum fits
    inside the D + G phases."""
    L = lib()
    cfg = L.config_init(1, seed=3, param_samples=64, events_per_sample=1024)
    cfg.phase_timing = 1
    ctx = make_ctx(cfg)
    for t in range(3):
        ctx.train_step(t, L.STEP_LOCAL_ONLY, _stream())
    ctx.timing_reset()
    for t in range(3, 6):
        ctx.train_step(t, L.STEP_LOCAL_ONLY, _stream())
    kt, n = ctx.kernel_times()
    ph, _ = ctx.phase_times()
    assert n == 3
    g_layers = ["g_fwd_first", "g_fwd_mid", "g_fwd_head", "g_bwd_last", "g_bwd_mid", "g_bwd_dy"]
    d_fwd = ["d_fwd_first", "d_fwd_mid", "d_fwd_head"]
    assert all(kt[k] > 0 for k in ["d_bwd_last", "d_bwd_mid", "d_bwd_first"]), kt
    assert all(kt[k] > 0 for k in d_fwd) or (kt["d_fwd_fused"] > 0 and all(kt[k] == 0 for k in d_fwd)), kt
    assert all(kt[k] > 0 for k in g_layers) or (kt["g_fused"] > 0 and all(kt[k] == 0 for k in g_layers)), kt
    assert sum(kt.values()) <= ph["disc_step"] + ph["gen_loss_through_disc"] + 1e-3


@pytest.mark.parametrize("preset", [0, 1])
def test_train_step_host_inputs_reproduce_the_device_step(preset):
    """sagips_train_step_host: the same step fed from pinned host memory with
    the noise and real rows the device RNG would have produced is bit-identical
    to the device-input step; the stats record arrives in the host buffer."""
    import ctypes
    L = lib()
    kw = dict(seed=21, param_samples=32, events_per_sample=45, reference_rows=4000, shard_rows=2000)
    ca, cb = make_ctx(L.config_init(preset, **kw)), make_ctx(L.config_init(preset, **kw))
    ca.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    torch.cuda.synchronize()
    N = 32 * 45
    noise = torch.from_numpy(ca.get(L.T_NOISE).reshape(32, -1).copy()).pin_memory()
    real = torch.from_numpy(ca.get(L.T_EVENTS).reshape(-1, 2)[:N].copy()).pin_memory()
    stats = (ctypes.c_uint8 * ctypes.sizeof(L.StepStats))()
    cb.train_step_host(0, L.STEP_LOCAL_ONLY, noise.data_ptr(), real.data_ptr(), ctypes.addressof(stats), _stream())
    torch.cuda.synchronize()
    for w in (L.T_NOISE, L.T_RAW, L.T_EVENTS, L.T_LOGITS_D, L.T_DISC_DW, L.T_DISC_DB, L.T_DY, L.T_DRAW, L.T_GEN_DW):
        assert np.array_equal(ca.get(w), cb.get(w)), w
    sa, sb = ca.get(L.T_STATS), L.StepStats.from_buffer_copy(stats)
    assert sa.loss_d == sb.loss_d and sa.loss_g == sb.loss_g and sb.nonfinite == 0
    # the real half of the histogram is zero (no bootstrap), the fake half as the device step
    ha, hb = ca.get(L.T_HIST).reshape(2, -1), cb.get(L.T_HIST).reshape(2, -1)
    assert np.all(hb[0] == 0) and np.array_equal(ha[1], hb[1])


def test_nonfinite_loss_is_reported():
    """The SPEC's NaN guard (include/sagips.h ERR_NONFINITE): a
    NaN in one discriminator weight makes both losses non-finite; the step's
    stats record carries the flag and reading it returns NONFINITE (after the
    copy), without aborting the process."""
    L = lib()
    ctx = make_ctx(L.config_init(1, seed=3, param_samples=32, events_per_sample=64))
    w = ctx.get(L.T_DISC_W)
    w[5] = np.nan
    ctx.set(L.T_DISC_W, w)
    ctx.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    with pytest.raises(L.SagipsError) as e:
        ctx.get(L.T_STATS)
    assert e.value.status == 4  # NONFINITE
    ctx.set(L.T_DISC_W, np.nan_to_num(w))  # the context stays usable
    ctx.train_step(1, L.STEP_LOCAL_ONLY, _stream())
    torch.cuda.synchronize()


@pytest.mark.parametrize("graph", [False, True])
def test_pipelined_host_input_steps_match_the_device_steps(graph):
    """sagips_train_step_host issued one step ahead (step t+1 before waiting
    for step t, as bench.py's e2e loop): the two staging slots and the copy
    stream keep every step's inputs apart -- six steps with distinct inputs
    end in the device-input run's parameters, bit for bit; also as CUDA-graph
    steps (the staged-input copies are memcpy nodes updated in place)."""
    import ctypes
    L = lib()
    kw = dict(seed=23, param_samples=32, events_per_sample=64, reference_rows=4000, shard_rows=2000)
    ca, cb = make_ctx(L.config_init(1, **kw)), make_ctx(L.config_init(1, **kw))
    N, T = 32 * 64, 6
    noises, reals = [], []
    for t in range(T):
        ca.train_step(t, 0, _stream())
        torch.cuda.synchronize()
        noises.append(torch.from_numpy(ca.get(L.T_NOISE).reshape(32, -1).copy()).pin_memory())
        reals.append(torch.from_numpy(ca.get(L.T_EVENTS).reshape(-1, 2)[:N].copy()).pin_memory())
    stats = [(ctypes.c_uint8 * ctypes.sizeof(L.StepStats))() for _ in range(T)]
    cur = torch.cuda.current_stream()
    done = [torch.cuda.Event() for _ in range(T)]
    for t in range(T):
        cb.train_step_host(t, L.STEP_GRAPH if graph else 0, noises[t].data_ptr(), reals[t].data_ptr(),
                           ctypes.addressof(stats[t]), _stream())
        done[t].record(cur)
        if t > 0:
            done[t - 1].synchronize()
    torch.cuda.synchronize()
    for w in (L.T_GEN_W, L.T_GEN_B, L.T_DISC_W, L.T_DISC_B):
        assert np.array_equal(ca.get(w), cb.get(w)), w
    sa, sb = ca.get(L.T_STATS), L.StepStats.from_buffer_copy(stats[T - 1])
    assert sa.loss_d == sb.loss_d and sa.loss_g == sb.loss_g


def _tabulated_cfg(L, preset, **kw):
    cfg = L.config_init(preset, seed=19, sampler=L.SAMPLER_TABULATED, sampler_grid=129, **kw)
    for j, v in enumerate((0.3, 2.0, 1.2, 0.7, 1.5, 3.0)):   # (w, b, c) per observable
        cfg.true_params[j] = v
    cfg.hist_lo[0] = cfg.hist_lo[1] = 0.0
    cfg.hist_hi[0] = cfg.hist_hi[1] = 1.0
    return cfg


@pytest.mark.parametrize("preset", [0, 1])
def test_tabulated_sampler_graph_and_host_inputs(preset):
    """The tabulated-CDF sampler (R32) through the other step paths: four
    CUDA-graph steps bit-identical to four eager ones, and a host-input step
    (the caller's noise and real rows) bit-identical to the device-input
    step it reproduces."""
    import ctypes
    L = lib()
    kw = dict(param_samples=32, events_per_sample=45, reference_rows=4000, shard_rows=2000)
    ca, cb = make_ctx(_tabulated_cfg(L, preset, **kw)), make_ctx(_tabulated_cfg(L, preset, **kw))
    for t in range(4):
        ca.train_step(t, 0, _stream())
        cb.train_step(t, L.STEP_GRAPH, _stream())
    torch.cuda.synchronize()
    for w in (L.T_GEN_W, L.T_GEN_B, L.T_DISC_W, L.T_DISC_B, L.T_EVENTS, L.T_DY, L.T_HIST):
        assert np.array_equal(ca.get(w), cb.get(w)), w
    cc = make_ctx(_tabulated_cfg(L, preset, **kw))
    cd = make_ctx(_tabulated_cfg(L, preset, **kw))
    cc.train_step(0, L.STEP_LOCAL_ONLY, _stream())
    torch.cuda.synchronize()
    N = 32 * 45
    noise = torch.from_numpy(cc.get(L.T_NOISE).reshape(32, -1).copy()).pin_memory()
    real = torch.from_numpy(cc.get(L.T_EVENTS).reshape(-1, 2)[:N].copy()).pin_memory()
    stats = (ctypes.c_uint8 * ctypes.sizeof(L.StepStats))()
    cd.train_step_host(0, L.STEP_LOCAL_ONLY, noise.data_ptr(), real.data_ptr(), ctypes.addressof(stats), _stream())
    torch.cuda.synchronize()
    for w in (L.T_RAW, L.T_EVENTS, L.T_LOGITS_D, L.T_DISC_DW, L.T_DY, L.T_DRAW, L.T_GEN_DW):
        assert np.array_equal(cc.get(w), cd.get(w)), w


@pytest.mark.parametrize("preset", [0, 1])
def test_graph_step_matches_eager(preset):
    """SAGIPS_STEP_GRAPH: the captured-and-replayed step runs
    the same kernels on the same inputs, so after several steps the parameters
    and losses are bit-identical to the eager step's; every step after the
    first is one graph launch, updated in place (one instantiation)."""
    L = lib()
    kw = dict(seed=17, param_samples=32, events_per_sample=64)
    ca, cb = make_ctx(L.config_init(preset, **kw)), make_ctx(L.config_init(preset, **kw))
    for t in range(5):
        ca.train_step(t, 0, _stream())
        cb.train_step(t, L.STEP_GRAPH, _stream())
    torch.cuda.synchronize()
    for w in (L.T_GEN_W, L.T_GEN_B, L.T_DISC_W, L.T_DISC_B, L.T_EVENTS, L.T_DY, L.T_HIST):
        assert np.array_equal(ca.get(w), cb.get(w)), w
    sa, sb = ca.get(L.T_STATS), cb.get(L.T_STATS)
    assert sa.loss_d == sb.loss_d and sa.loss_g == sb.loss_g
    launches, inst = cb.graph_stats()
    assert launches == 4 and inst == 1, (launches, inst)
