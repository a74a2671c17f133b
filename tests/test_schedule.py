"""Schedule from measured B200 constants: the restated
build_schedule (schedule.hpp:177-209) against the compiled reference on random
and calibrated operator sets, and the measured-constant plumbing."""
import json

import numpy as np
import pytest

from paper_2412_15411_b200 import schedule as S


def ops_dicts(ops):
    return [dict(cls=o.cls, params=o.params, hard=o.hard, soft=o.soft, ema=o.ema, capacity=o.capacity) for o in ops]


def random_ops(rng, n):
    ops = []
    for i in range(n):
        cls = int(rng.choice([S.EXPERT, S.EXPERT, S.EXPERT, S.NON_EXPERT, S.GATE]))
        ops.append(S.Operator(i, cls, int(rng.integers(1, 5_000_000)),
                              hard=float(rng.integers(0, 6)),  # ties on purpose
                              soft=float(rng.random()), ema=float(rng.random()),
                              capacity=float(rng.integers(1, 4))))
    return ops


def check_same(reference, ops, plan, bw, t_iter, ordering=S.HARD, allow_single=False):
    from oracle.oracle import ref_build_schedule
    try:
        ref = ref_build_schedule(reference, ops_dicts(ops), plan.compute_bytes, plan.master_bytes,
                                 plan.optimizer_bytes, bw, t_iter, ordering, allow_single)
    except RuntimeError as e:
        # the reference overruns its operator list when the grown window's
        # last slot starts past the end (std::length_error); so must we
        assert "max_size" in str(e)
        with pytest.raises(ValueError, match="past the"):
            S.build_schedule(ops, plan, bw, t_iter, ordering, allow_single)
        return False
    got = S.build_schedule(ops, plan, bw, t_iter, ordering, allow_single)
    w, o, fits, slots = ref
    assert (got.wsparse, got.o_active, got.fits_budget) == (w, o, fits)
    assert [(list(a), list(c)) for a, c in got.slots] == slots
    return True


@pytest.mark.parametrize("seed", range(12))
def test_build_schedule_matches_reference_random(reference, seed):
    rng = np.random.default_rng(seed)
    ops = random_ops(rng, int(rng.integers(1, 60)))
    plan = S.Precision(int(rng.choice([1, 2, 4])), 4, 8)
    total = sum(o.params for o in ops) * plan.full_state_bytes
    # budgets from "everything fits" down to "even the floor stalls"
    same = 0
    for frac in (2.0, 0.5, 0.2, 0.05, 0.001):
        for ordering in (S.HARD, S.SOFT, S.DECAY, S.CAPACITY):
            same += check_same(reference, ops, plan, total * frac, 1.0, ordering, allow_single=bool(seed % 2))
    assert same  # most budgets produce a schedule


def test_deepseek_profile_matches_reference_and_survey(reference):
    """configs/deepseek_moe.json under its own PCIe constant: W=6, O=368
    (SURVEY.md 8(a) a20), identical to the reference; then the measured ones."""
    pop = [(e % 64 + 1) ** -0.5 for e in range(28 * 64)]
    ops = S.deepseek_layer_ops(28, popularity=pop)
    t_iter = S.iteration_time([0.12] * 12, 16, 0.1405, 0.074)
    s = S.build_schedule(ops, S.Precision(), 18.95e9, t_iter)
    assert (s.wsparse, s.o_active) == (6, 368)
    check_same(reference, ops, S.Precision(), 18.95e9, t_iter)
    for bw in (54e9, 645e9):
        check_same(reference, ops, S.Precision(), bw, t_iter)


def test_measured_constants_shrink_the_window():
    line = json.dumps({"unit": "GB/s", "value": 1290.0, "n_gpus": 2, "e2e": {"value": 54.0, "unit": "GB/s"}})
    m = S.Measured.from_bench(line)
    assert m.host == pytest.approx(54e9) and m.device == pytest.approx(645e9)
    pop = [(e % 64 + 1) ** -0.5 for e in range(28 * 64)]
    res = S.compare(S.deepseek_layer_ops(28, popularity=pop), S.Precision(),
                    S.iteration_time([0.12] * 12, 16, 0.1405, 0.074), 18.95e9, m)
    w = [res[k]["wsparse"] for k in ("reference_pcie", "b200_host", "b200_device")]
    assert w == sorted(w, reverse=True) and w[0] == 6 and w[-1] >= 1
    assert res["b200_host"]["recovery_s_expected"] < res["reference_pcie"]["recovery_s_expected"]


def test_schedule_errors():
    with pytest.raises(ValueError, match="non-positive budget"):
        S.find_window_size(4, 1.0, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError, match="no operators"):
        S.build_schedule([], S.Precision(), 1.0, 1.0)
    with pytest.raises(ValueError, match="has no capacity"):
        S.order_operators([S.Operator(0, S.EXPERT, 10)], S.CAPACITY)
