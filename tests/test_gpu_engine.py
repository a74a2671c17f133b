"""The GPU toy trainer (mlck_engine) against the reference:
run_iteration's next state, weight gradients and boundary log; the
recompute-replay conversion and localized recovery.

Tolerance (stated: recompute parity is tolerance-based).  The
forward calls tanh and exp.  The GPU evaluates them in double and rounds once
(the correctly rounded tanhf / expf); the reference calls glibc's tanhf
(expm1f-based, not correctly rounded) and expf.  Everything else -- operation
order, the canonical (replica, micro-batch, token) summation, no FMA -- is
the reference's, so the two differ by the ulps of those calls as they
propagate: measured max normalized error ~1e-7.  Asserted per array:
max|gpu - ref| <= RTOL * max|ref| (RTOL = 1e-5), and routing, steps, stages
and boundary-log keys identical."""
import numpy as np
import pytest

from golden_cases import load_case
from oracle.oracle import RefEngine, ref_convert, toy_config

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(scope="module")
def mk():
    from paper_2412_15411_b200 import mlck
    return mlck


@pytest.fixture(scope="module")
def ctx(mk):
    c = mk.Context(0)
    yield c
    c.close()


def nerr(a, b):
    """max |a - b| / max |b| (normalized max error of float32 arrays)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if not b.size:
        return 0.0
    scale = np.max(np.abs(b))
    d = np.max(np.abs(a - b))
    return float(d / scale) if scale > 0 else float(d)


def upload(mk, ctx, c, s):
    st = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    for i in range(c.n_ops):
        o = c.op(s, i)
        st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
    st.set_meta(s, c.data_seed)
    return st


CASES = ["verify_toy", "dp2_pp2", "six_op_cb1", "toy_sgd"]


@pytest.mark.parametrize("name", CASES)
def test_run_iteration_matches_reference(mk, ctx, name):
    """Engine::run_iteration from every golden state: the next state, the
    iteration's weight gradients (zero-copy into the gradient log) and the
    sender-side boundary entries."""
    c = load_case(name)
    eng = mk.Engine(ctx, c.meta["cfg"])
    assert eng.param_counts() == c.meta["param_counts"]
    assert [eng.stage_of_op(i) for i in range(c.n_ops)] == c.meta["stage_of_op"]
    worst = 0
    log = mk.UpstreamLog(ctx, 1 << 24, kind=0)
    g = mk.GradLog(ctx, c.meta["param_counts"], c.T + 1)
    for s in range(c.T):
        st = upload(mk, ctx, c, s)
        eng.run_iteration(st, log=log, gradlog=g)
        assert st.meta() == (s + 1, c.data_seed)
        for i in range(c.n_ops):
            got, want = st.download_op(i), c.op(s + 1, i)
            assert got.step == want["step"]
            for x, y in ((got.master, want["master"]), (got.m, want["m"]), (got.v, want["v"])):
                worst = max(worst, nerr(x, y))
            gd = np.frombuffer(ctx.download(g.slot(s + 1, i), 4 * c.meta["param_counts"][i]), np.float32)
            worst = max(worst, nerr(gd, c.grads(s + 1, i)))
        st.close()
    assert worst <= RTOL, worst
    want = {k: v for k, v in c.log_entries()} if "log_keys" in c.d else {}
    got = dict(log.entries())
    if want:
        assert sorted(got) == sorted(want)
        for k in want:
            assert nerr(got[k], want[k]) <= RTOL, k


@pytest.mark.parametrize("name", ["verify_toy", "dp2_pp2", "six_op_cb1"])
def test_recompute_conversion_matches_reference(mk, ctx, name):
    """sparse_to_dense_convert by recompute (frozen operators: input gradients
    only) == the reference's conversion of the same window."""
    c = load_case(name)
    eng = mk.Engine(ctx, c.meta["cfg"])
    for w in c.meta["converted_windows"]:
        blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
        out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
        eng.sparse_to_dense_convert(out, blobs, w, c.W, c.data_seed)
        got, want = out.serialize_state(), c.converted(w)
        if got != want:  # within the tanh / exp tolerance
            assert len(got) == len(want)
            hdr = 28
            assert got[:hdr] == want[:hdr]
            worst = 0
            pos = hdr
            for P in c.meta["param_counts"]:
                assert got[pos:pos + 16] == want[pos:pos + 16]
                for j in range(3):  # master, m, v
                    a = np.frombuffer(got, np.float32, P, pos + 16 + 4 * P * j)
                    b = np.frombuffer(want, np.float32, P, pos + 16 + 4 * P * j)
                    worst = max(worst, nerr(a, b))
                pos += 16 + 12 * P
            assert worst <= RTOL, (w, worst)


def test_recompute_localized_recovery_matches_reference(mk, ctx):
    """localized_recover by recompute: the segment's stages only, boundary
    tensors from the reference's own log."""
    c = load_case("dp2_pp2")
    eng = mk.Engine(ctx, c.meta["cfg"])
    log = mk.UpstreamLog(ctx, 1 << 24, kind=1, device=0)
    bufs = []
    for (it, mb, b, d), data in c.log_entries():
        p = ctx.upload(np.ascontiguousarray(data, np.float32))
        bufs.append(p)
        log.put(it, mb, b, d, p, data.size)
    log.sync()
    for (w, target, lo, hi) in c.localized():
        blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
        out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
        eng.localized_recover(out, lo, hi, blobs, w, c.W, c.data_seed, log, target)
        it, ref = c.localized_image(w, target, lo, hi)
        assert out.meta()[0] == it
        worst = 0
        for i in c.scope(lo, hi):
            step, master, m, v = ref[i]
            got = out.download_op(i)
            assert got.step == step
            for x, y in ((got.master, master), (got.m, m), (got.v, v)):
                worst = max(worst, nerr(x, y))
        assert worst <= RTOL, (w, target, lo, hi, worst)
    for p in bufs:
        ctx.free(p)


def test_recompute_errors(mk, ctx):
    c = load_case("verify_toy")
    eng = mk.Engine(ctx, c.meta["cfg"])
    blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(3)]
    out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    with pytest.raises(RuntimeError, match="sparse checkpoint incomplete: 2 of 3 records"):
        eng.sparse_to_dense_convert(out, blobs[:2], 3, 3, c.data_seed)
    with pytest.raises(RuntimeError, match="conversion finished with frozen operator"):
        eng.sparse_to_dense_convert(out, [blobs[0], blobs[1], blobs[1]], 3, 3, c.data_seed)
    empty = mk.UpstreamLog(ctx, 1 << 16, kind=0)
    with pytest.raises(RuntimeError, match="upstream log missing entry: iteration 4 micro-batch 0 boundary 0 fwd"):
        eng.localized_recover(out, 1, 1, blobs, 3, 3, c.data_seed, empty, 6)
    with pytest.raises(ValueError, match="top_k"):
        mk.Engine(ctx, dict(c.meta["cfg"], top_k=9))


def test_engine_at_configs0_scale_matches_reference(mk, ctx, reference):
    """8 experts + NE + G of 2^21 parameters (configs[0]): two reference
    iterations, every parameter (the toy model reads the first few, Adam
    moves all of them)."""
    P = 1 << 21
    cfg = toy_config(layers=1, experts=8, top_k=2, expert_params=P, nonexpert_params=P, gate_params=P, seed=3)
    ref = RefEngine(reference, cfg)
    eng = mk.Engine(ctx, dict(layers=1, experts_per_layer=8, top_k=2, shared_experts=0, token_dim=4,
                              expert_hidden=4, nonexpert_hidden=4, residual=1, expert_params=P, nonexpert_params=P,
                              gate_params=P, pp_stages=1, dp_degree=1, microbatches=2, microbatch_size=4,
                              compute_bytes=2))
    st = mk.DeviceState(ctx, [P] * 10, 2)
    state = ref.state()
    for i, op in enumerate(state.ops):
        st.upload_op(i, op.master, op.m, op.v, op.step)
    st.set_meta(ref.iteration, ref.data_seed)
    for _ in range(2):
        ref.run_iteration()
        eng.run_iteration(st)
    worst = 0
    for i, op in enumerate(ref.state().ops):
        got = st.download_op(i)
        assert got.step == op.step
        for x, y in ((got.master, op.master), (got.m, op.m), (got.v, op.v)):
            worst = max(worst, nerr(x, y))
    assert worst <= RTOL, worst


@pytest.mark.parametrize("name", ["verify_toy", "dp2_pp2"])
def test_gpu_run_window_replays_bit_exact(mk, ctx, name):
    """A window captured from the GPU trainer's own run: its records taken
    the reference's way (capture_windows), its weight gradients landing in the
    gradient log with no copy.  Both conversions -- recompute replay and
    logged-gradient replay -- rebuild the run's state bit for bit."""
    c = load_case(name)
    eng = mk.Engine(ctx, c.meta["cfg"])
    P, W = c.meta["param_counts"], c.W
    st = upload(mk, ctx, c, W)  # window [W, 2W)
    g = mk.GradLog(ctx, P, W + 1)
    blobs = []
    for k in range(W):
        blobs.append(mk.snapshot_record(st, *c.slot(k), k, 1, W, W))
        eng.run_iteration(st, gradlog=g)
    want = st.serialize_state()
    out = mk.DeviceState(ctx, P, c.compute_bytes)
    eng.sparse_to_dense_convert(out, blobs, W, W, c.data_seed)
    assert out.serialize_state() == want
    out2 = mk.DeviceState(ctx, P, c.compute_bytes)
    o = c.optimizer
    mk.sparse_to_dense_convert(out2, blobs, W, W, c.data_seed, g,
                               mk.Optimizer(o["kind"], o["lr"], o["beta1"], o["beta2"], o["eps"]))
    assert out2.serialize_state() == want
