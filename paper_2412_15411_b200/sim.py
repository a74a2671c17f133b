"""ETTR of the sparse-checkpoint policy under measured B200 constants
(second half).

The reference turns a cluster's constants into an effective-training-time
ratio with a discrete-event simulation (run_simulation, sim.hpp:246-597):
every iteration may stall on its snapshot (bytes / pcie_bandwidth beyond
t_iter), records drain to their replicas through a FIFO pipe
(replication_bandwidth x replication_r), failures arrive as a Poisson
process, and a failure rolls the failed pipeline segment back to the newest
persisted window, replays it (localized, from the boundary logs) and catches
up.  This module restates the policy this repository implements -- the
sparse (MoEtion) policy with Poisson failures -- so it can run on the
bandwidths bench.py measures on B200, and `tests/test_sim.py` pins it to the
compiled reference's own run_simulation on random configurations (equal
metrics to the last bit: same xoshiro streams, same IEEE operations).

Host-side policy arithmetic (no device work), so plain Python.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

from .schedule import EXPERT, GATE, HARD, NON_EXPERT, Operator, Precision, build_schedule

MASK = (1 << 64) - 1


class Rng:
    """xoshiro256++ with the reference's named substreams (rng.hpp:14-106)."""

    def __init__(self, seed: int):
        x = seed & MASK
        self.s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & MASK
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
            self.s.append(z ^ (z >> 31))

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & MASK

    def next_u64(self) -> int:
        s = self.s
        r = (self._rotl((s[0] + s[3]) & MASK, 23) + s[0]) & MASK
        t = (s[1] << 17) & MASK
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return r

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform_index(self, n: int) -> int:
        return 0 if n == 0 else self.next_u64() % n

    def exponential(self, mean: float) -> float:
        return -mean * math.log1p(-self.uniform())

    def substream(self, label: str, index: int = 0) -> "Rng":
        h = 0xCBF29CE484222325
        for v in list(label.encode()) + [index & MASK, self.s[0], self.s[2]]:
            h ^= v
            h = (h * 0x100000001B3) & MASK
        return Rng(h)


@dataclass
class SimConfig:
    """The SimConfig fields the sparse policy reads (sim.hpp:158-175; core.hpp)."""
    layers: int = 1
    experts_per_layer: int = 8
    expert_params: int = 1 << 20
    nonexpert_params: int = 1 << 20
    gate_params: int = 1 << 10
    tokens_per_sample: int = 1
    precision: Precision = field(default_factory=Precision)
    nodes: int = 1
    pcie_bandwidth: float = 1e10
    replication_bandwidth: float = 1e11
    pp_stages: int = 1
    microbatches: int = 1
    global_batch: int = 1
    t_stage: list = field(default_factory=lambda: [1.0])
    t_sync: float = 0.0
    t_update: float = 0.0
    t_iter_override: float = 0.0
    ordering: int = HARD
    upstream_logging: bool = True
    conversion_compute_savings: bool = False
    mtbf: float = 3600.0
    horizon: float = 3600.0
    t_restart: float = 30.0
    detection_delay: float = 5.0
    replication_r: int = 2
    seed: int = 1

    def operators(self) -> list[Operator]:
        """ModelSpec::operators (core.hpp:105-134): zero popularity."""
        ops = []
        for _ in range(self.layers):
            for _ in range(self.experts_per_layer):
                ops.append(Operator(len(ops), EXPERT, self.expert_params))
            ops.append(Operator(len(ops), NON_EXPERT, self.nonexpert_params))
            ops.append(Operator(len(ops), GATE, self.gate_params))
        return ops

    def iteration_time(self) -> float:
        """iteration_time (sim.hpp:35-47)."""
        if self.t_iter_override > 0:
            return self.t_iter_override
        return (self.microbatches + len(self.t_stage) - 1) * max(self.t_stage) + self.t_sync + self.t_update


def run_simulation(cfg: SimConfig) -> dict:
    """run_simulation (sim.hpp:246-597) for PolicyKind::Sparse and Poisson failures."""
    ops = cfg.operators()
    t_iter = cfg.iteration_time()
    if t_iter <= 0:
        raise ValueError("simulation: t_iter must be > 0")
    pcie = cfg.pcie_bandwidth
    stages = cfg.pp_stages
    sched = build_schedule(ops, cfg.precision, pcie, t_iter, cfg.ordering)
    slot_bytes = [sched.slot_bytes(i, ops, cfg.precision) for i in range(len(sched.slots))]
    rng = Rng(cfg.seed)
    victim_rng = rng.substream("victims")
    failure_rng = rng.substream("failures")

    pipe_tail = 0.0  # DrainQueue (sim.hpp:215-223)
    pending, persisted_state = [(0, 0.0)], 0  # PersistedTracker (sim.hpp:225-238)

    def push(ready, nbytes):
        nonlocal pipe_tail
        pipe_tail = max(pipe_tail, ready) + nbytes / cfg.replication_bandwidth
        return pipe_tail

    def frontier(now):
        nonlocal persisted_state
        while pending and pending[0][1] <= now:
            persisted_state = max(persisted_state, pending[0][0])
            pending.pop(0)
        return persisted_state

    def replay_cost(lo, hi):
        if not cfg.upstream_logging or not cfg.t_stage:
            return t_iter
        worst = max(cfg.t_stage[lo:hi + 1])
        return (cfg.microbatches + (hi - lo + 1) - 1) * worst + cfg.t_update

    def discount():
        if not cfg.conversion_compute_savings:
            return 1.0
        w = sched.wsparse
        share = 0.0
        for k in range(w):
            share += (w - 1 - k) / w
        share /= w
        return 1.0 - share / 3.0

    next_poisson = failure_rng.exponential(cfg.mtbf)
    useful = stall_total = recovery_total = idle_total = 0.0
    state, wall, iterations, failures = 0, 0.0, 0, 0
    recompute_total = max_event = mean_event = 0.0
    never = False
    while wall < cfg.horizon:
        k = state + 1
        snap_bytes = slot_bytes[state % sched.wsparse]
        snap_time = snap_bytes / pcie if snap_bytes > 0 else 0.0
        stall_k = max(0.0, snap_time - t_iter)
        t_eff = t_iter + stall_k
        fail_at, fail_node = math.inf, -1
        if next_poisson < wall + t_eff and next_poisson < fail_at:
            fail_at = next_poisson
            fail_node = victim_rng.uniform_index(max(cfg.nodes, 1))
        if fail_at >= wall + t_eff:  # clean iteration
            wall += t_eff
            useful += t_iter
            stall_total += stall_k
            state = k
            iterations += 1
            if snap_bytes > 0:
                pending.append((state - 1, push(wall, snap_bytes * cfg.replication_r)))
            continue
        failures += 1
        partial = fail_at - wall
        recovery_total += partial
        event = partial
        wall = fail_at
        seg = fail_node % stages if stages > 0 else 0
        idle_total += cfg.detection_delay + cfg.t_restart
        wall += cfg.detection_delay + cfg.t_restart
        f = frontier(wall)
        w = sched.wsparse
        a = (f - (w - 1)) // w * w if f >= w - 1 else -1
        if a < 0:  # no complete window yet: global restart
            recompute = float(state) * t_iter
            never = True
            resume = state
        else:
            target = a + w
            catchup = max(0, state - target)
            recompute = (w + catchup) * (replay_cost(seg, seg) * discount())
            resume = max(state, target)
        recovery_total += recompute
        event += recompute
        recompute_total += recompute
        wall += recompute
        state = resume
        max_event = max(max_event, event)
        mean_event += event
        next_poisson = wall + failure_rng.exponential(cfg.mtbf)
    if failures:
        mean_event /= failures
    wall_s = useful + stall_total + recovery_total + idle_total
    return {"wsparse": sched.wsparse, "t_iter": t_iter, "iterations": iterations, "failures": failures,
            "useful_s": useful, "stall_s": stall_total, "recovery_s": recovery_total, "idle_s": idle_total,
            "wall_s": wall_s, "ettr": useful / wall_s if wall_s > 0 else 1.0,
            "overhead_s_per_iter": stall_total / iterations if iterations else 0.0,
            "recovery_recompute_s": recompute_total, "max_recovery_event_s": max_event,
            "mean_recovery_event_s": mean_event, "checkpoint_never_persisted": never}


def deepseek_config(**kw) -> SimConfig:
    """configs/deepseek_moe.json with its sim block (mtbf 600 s, 12 h)."""
    base = dict(layers=28, experts_per_layer=64, expert_params=7_898_100, nonexpert_params=80_140_000,
                gate_params=100_000, tokens_per_sample=2048, nodes=12, pcie_bandwidth=18.95e9,
                replication_bandwidth=1e12, pp_stages=12, microbatches=16, global_batch=512, t_stage=[0.12] * 12,
                t_sync=0.1405, t_update=0.074, mtbf=600.0, horizon=43200.0, t_restart=10.0, detection_delay=2.0,
                replication_r=2, seed=7)
    base.update(kw)
    return SimConfig(**base)


def _main():
    import argparse
    ap = argparse.ArgumentParser(description="ETTR of configs/deepseek_moe.json under the reference's constants "
                                             "and the B200 constants of a bench.py line")
    ap.add_argument("bench_json", help="file holding a bench.py JSON line (N=1 and/or N>1)")
    args = ap.parse_args()
    lines = [json.loads(x) for x in open(args.bench_json).read().splitlines() if x.strip().startswith("{")]
    j = lines[-1]
    host = float(j["e2e"]["value"]) * 1e9                       # record to pinned host (the PCIe analogue)
    dev = float(j["value"]) / max(1, int(j.get("n_gpus", 1))) * 1e9  # on-device snapshot + replica per GPU
    out = {}
    for name, kw in (("reference", {}),
                     ("b200_host", dict(pcie_bandwidth=host)),
                     ("b200_device", dict(pcie_bandwidth=dev, replication_bandwidth=dev))):
        out[name] = run_simulation(deepseek_config(**kw))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    _main()
