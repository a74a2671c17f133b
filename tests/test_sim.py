"""paper_2412_15411_b200.sim (run_simulation's sparse policy)
pinned to the compiled reference's run_simulation (sim.hpp:246-597): every
metric equal, on random cluster / model / failure configurations and on
configs/deepseek_moe.json under the reference's and B200-measured constants."""
import ctypes as C

import numpy as np
import pytest

from paper_2412_15411_b200 import sim

FIELDS = ["wsparse", "t_iter", "iterations", "failures", "useful_s", "stall_s", "recovery_s", "idle_s", "wall_s",
          "ettr", "overhead_s_per_iter", "recovery_recompute_s", "max_recovery_event_s", "mean_recovery_event_s",
          "checkpoint_never_persisted"]


def ref_run(reference, cfg: sim.SimConfig) -> dict:
    L = reference.lib
    f = L.mlr_run_simulation_sparse
    f.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_double,
                  C.c_double, C.c_int32, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.c_int32, C.c_double,
                  C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                  C.c_int32, C.c_uint64, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    ts = (C.c_double * len(cfg.t_stage))(*cfg.t_stage)
    out = (C.c_double * len(FIELDS))()
    err = C.create_string_buffer(512)
    rc = f(cfg.layers, cfg.experts_per_layer, cfg.expert_params, cfg.nonexpert_params, cfg.gate_params,
           cfg.tokens_per_sample, cfg.nodes, cfg.pcie_bandwidth, cfg.replication_bandwidth, cfg.pp_stages,
           cfg.microbatches, cfg.global_batch, ts, len(cfg.t_stage), cfg.t_sync, cfg.t_update, cfg.t_iter_override,
           int(cfg.upstream_logging), int(cfg.conversion_compute_savings), cfg.mtbf, cfg.horizon, cfg.t_restart,
           cfg.detection_delay, cfg.replication_r, cfg.seed, out, err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return dict(zip(FIELDS, list(out)))


def same(ours: dict, ref: dict):
    for k in FIELDS:
        a, b = float(ours[k]), float(ref[k])
        assert a == b, (k, a, b)


def random_configs():
    rng = np.random.default_rng(3)
    out = []
    for i in range(30):
        stages = int(rng.integers(1, 9))
        out.append(sim.SimConfig(
            layers=int(rng.integers(stages, 12)), experts_per_layer=int(rng.integers(2, 65)),
            expert_params=int(rng.integers(1, 10 ** 7)), nonexpert_params=int(rng.integers(1, 10 ** 8)),
            gate_params=int(rng.integers(1, 10 ** 5)), nodes=int(rng.integers(1, 17)),
            pcie_bandwidth=float(rng.uniform(1e9, 1e12)), replication_bandwidth=float(rng.uniform(1e9, 1e13)),
            pp_stages=stages, microbatches=int(rng.integers(1, 33)), global_batch=64,
            t_stage=[float(x) for x in rng.uniform(0.01, 0.5, stages)], t_sync=float(rng.uniform(0, 0.2)),
            t_update=float(rng.uniform(0, 0.1)), upstream_logging=bool(i % 3), conversion_compute_savings=bool(i % 2),
            mtbf=float(rng.uniform(30, 3000)), horizon=float(rng.uniform(600, 20000)),
            t_restart=float(rng.uniform(0, 30)), detection_delay=float(rng.uniform(0, 5)),
            replication_r=int(rng.integers(1, 4)), seed=int(rng.integers(1, 2 ** 62))))
    return out


def test_rng_matches_reference_streams(reference):
    """xoshiro256++ + substreams: the failure gaps the reference draws."""
    cfg = sim.SimConfig(mtbf=100.0, horizon=5000.0, seed=11)
    ours, ref = sim.run_simulation(cfg), ref_run(reference, cfg)
    assert ours["failures"] == ref["failures"] > 5
    same(ours, ref)


@pytest.mark.parametrize("i", range(30))
def test_random_configs_match_reference(reference, i):
    cfg = random_configs()[i]
    try:
        ref = ref_run(reference, cfg)
    except RuntimeError as e:
        with pytest.raises(Exception, match=str(e)[:30]):
            sim.run_simulation(cfg)
        return
    same(sim.run_simulation(cfg), ref)


@pytest.mark.parametrize("pcie", [18.95e9, 56e9, 830e9])
def test_deepseek_profile_matches_reference(reference, pcie):
    """configs/deepseek_moe.json (28 layers, mtbf 600 s, 12 h) at the
    reference's PCIe figure and at the B200 host / device rates."""
    cfg = sim.deepseek_config(pcie_bandwidth=pcie, horizon=7200.0)
    same(sim.run_simulation(cfg), ref_run(reference, cfg))
