"""Host-side entry points of the drop-in boundary, on CPU: the log storage
budget (recovery.hpp:296-317) against the compiled reference, and the
header's new entries in the ABI (no GPU needed for any of these)."""
import itertools

import numpy as np
import pytest

from oracle.oracle import RefError, ref_check_log_budget, toy_config


@pytest.fixture(scope="module")
def mk():
    from paper_2412_15411_b200 import mlck
    return mlck


def configs():
    rng = np.random.default_rng(11)
    out = [dict(token_dim=2048, stages=4, micro=8, mb=4096, dp=2, w=6)]  # configs[4]
    for _ in range(40):
        out.append(dict(token_dim=int(rng.integers(1, 8192)), stages=int(rng.integers(1, 9)),
                        micro=int(rng.integers(1, 17)), mb=int(rng.integers(1, 4097)),
                        dp=int(rng.integers(1, 5)), w=int(rng.integers(1, 9))))
    return out


@pytest.mark.parametrize("c", configs())
def test_upstream_log_bytes_matches_reference(mk, reference, c):
    ref = reference
    cfg = toy_config(layers=max(8, c["stages"]), stages=c["stages"], token_dim=c["token_dim"],
                     microbatches=c["micro"], mb_size=c["mb"], dp=c["dp"])
    want = ref.lib.mlr_upstream_log_bytes(cfg, c["w"])
    got = mk.upstream_log_bytes(c["token_dim"], c["stages"], c["micro"], c["mb"], c["dp"], c["w"])
    assert got == want


def test_upstream_log_bytes_baseline_config(mk):
    # configs[4]: dp2 x pp4, M=8, [4096 x 2048] f32, W=6 -> 38.65 GB
    assert mk.upstream_log_bytes(2048, 4, 8, 4096, 2, 6) == 38_654_705_664


@pytest.mark.parametrize("mem,nodes", list(itertools.product([0.0, -1.0, 1e6, 4e9, 1e12], [1, 3])))
def test_check_log_budget_matches_reference(mk, reference, mem, nodes):
    ref = reference
    cfg = toy_config(layers=8, stages=4, token_dim=512, microbatches=4, mb_size=256, dp=2)
    want = None
    try:
        ref_check_log_budget(ref, cfg, 5, mem, nodes)
    except RefError as e:
        want = str(e)
    if want is None:
        mk.check_log_budget(512, 4, 4, 256, 2, 5, mem, nodes)
    else:
        with pytest.raises(ValueError) as ei:  # std::invalid_argument
            mk.check_log_budget(512, 4, 4, 256, 2, 5, mem, nodes)
        assert str(ei.value) == want
