"""Sparse-checkpoint schedule fed by measured B200 constants.

The reference sizes its window from a budget of `pcie_bandwidth * t_iter`
bytes per iteration (build_schedule, schedule.hpp:177-209): the smallest
window whose per-iteration snapshot fits in one iteration.  Its configs carry
a PCIe figure from other hardware (configs/deepseek_moe.json: 18.95 GB/s).
This module restates the policy -- operator ordering, window sizing, slot
generation and the exact-size validation -- so it can run on the bandwidth
this repository measures on B200 (`bench.py`'s JSON line), and reports what
that does to W and to the recovery-time bounds (recovery.hpp:328-334).

Host-side and microsecond-scale (the schedule is rebuilt on popularity
drift, not per iteration), so plain Python; tests pin it to the compiled
reference's build_schedule on random and calibrated operator sets.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

EXPERT, NON_EXPERT, GATE = 0, 1, 2          # OperatorClass (core.hpp:33-37)
HARD, SOFT, DECAY, CAPACITY = 0, 1, 2, 3    # OrderingScheme (schedule.hpp:16-21)


@dataclass
class Operator:
    """OperatorDescriptor (core.hpp:41-61): the fields the schedule reads."""
    id: int
    cls: int = EXPERT
    params: int = 0
    hard: float = 0.0
    soft: float = 0.0
    ema: float = 0.0
    capacity: float = 0.0


@dataclass
class Precision:
    """PrecisionPlan (core.hpp:16-27)."""
    compute_bytes: int = 2
    master_bytes: int = 4
    optimizer_bytes: int = 8

    @property
    def full_state_bytes(self) -> int:
        return self.master_bytes + self.optimizer_bytes


@dataclass
class Schedule:
    wsparse: int
    o_active: int
    ordering: int
    fits_budget: bool
    slots: list = field(default_factory=list)  # [(active ids, compute-only ids)]

    def slot_bytes(self, i: int, ops: list[Operator], plan: Precision) -> int:
        """SparseSchedule::slot_bytes (schedule.hpp:128-136)."""
        a, c = self.slots[i]
        return sum(ops[j].params * plan.full_state_bytes for j in a) + sum(ops[j].params * plan.compute_bytes for j in c)

    def max_slot_bytes(self, ops: list[Operator], plan: Precision) -> int:
        return max((self.slot_bytes(i, ops, plan) for i in range(len(self.slots))), default=0)


def order_operators(ops: list[Operator], scheme: int) -> list[int]:
    """Ascending popularity, ties by id; non-experts and gates after all
    experts in id order (schedule.hpp:41-80)."""
    def score(op: Operator) -> float:
        if scheme == HARD:
            return op.hard
        if scheme == SOFT:
            return op.soft
        if scheme == DECAY:
            return op.ema
        if op.capacity <= 0:
            raise ValueError(f"capacity-aware ordering: operator {op.id} has no capacity")
        return op.hard / op.capacity

    experts = sorted((op for op in ops if op.cls == EXPERT), key=lambda op: (score(op), op.id))
    rest = sorted(op.id for op in ops if op.cls != EXPERT)
    return [op.id for op in experts] + rest


def find_window_size(o_total: int, mean_full: float, mean_compute: float, bandwidth: float, t_iter: float,
                     allow_single: bool = False) -> tuple[int, int, bool]:
    """Freeze operators one at a time until the per-iteration snapshot fits
    the budget (schedule.hpp:92-118).  Returns (wsparse, o_active, fits)."""
    if bandwidth <= 0 or t_iter <= 0:
        raise ValueError("find_window_size: non-positive budget")
    if o_total <= 0:
        raise ValueError("find_window_size: no operators")
    budget = bandwidth * t_iter
    floor_active = 1 if allow_single else 2
    o_active = o_total
    while o_active > floor_active:
        if mean_full * o_active + mean_compute * (o_total - o_active) <= budget:
            break
        o_active -= 1
    fits = mean_full * o_active + mean_compute * (o_total - o_active) <= budget
    return (o_total + o_active - 1) // o_active, o_active, fits


def generate_schedule(ordered: list[int], wsparse: int, o_active: int, ordering: int) -> Schedule:
    """Slot i: ordered[i*O : (i+1)*O] active, everything after compute-only
    (schedule.hpp:153-172)."""
    if not ordered:
        raise ValueError("generate_schedule: empty operator list")
    n = len(ordered)
    s = Schedule(wsparse, o_active, ordering, True)
    for i in range(wsparse):
        start = i * o_active
        end = min(start + o_active, n)
        if start > n:  # the reference's vector::assign(begin + start, begin + end) throws length_error
            raise ValueError(f"generate_schedule: slot {i} starts at operator {start} past the {n} operators")
        s.slots.append((ordered[start:end], ordered[end:]))
    return s


def build_schedule(ops: list[Operator], plan: Precision, bandwidth: float, t_iter: float, ordering: int = HARD,
                   allow_single: bool = False) -> Schedule:
    """Mean-size window search, ordering, then exact-size validation that grows
    the window until every slot fits (schedule.hpp:177-209)."""
    n = len(ops)
    if n == 0:
        raise ValueError("find_window_size: no operators")
    total_full = sum(float(op.params * plan.full_state_bytes) for op in ops)
    total_compute = sum(float(op.params * plan.compute_bytes) for op in ops)
    wsparse, o_active, fits = find_window_size(n, total_full / n, total_compute / n, bandwidth, t_iter, allow_single)
    ordered = order_operators(ops, ordering)
    budget = bandwidth * t_iter
    while True:
        sched = generate_schedule(ordered, wsparse, o_active, ordering)
        sched.fits_budget = fits
        if float(sched.max_slot_bytes(ops, plan)) <= budget:
            break
        if o_active <= (1 if allow_single else 2) or wsparse >= n:
            sched.fits_budget = False  # checkpointing will stall
            break
        wsparse += 1
        o_active = (n + wsparse - 1) // wsparse
    return sched


def recovery_time_bounds_sparse(wsparse: float, t_iter: float) -> tuple[float, float, float]:
    """(min, max, expected) recovery time (recovery.hpp:328-330)."""
    return 0.0, 2.0 * wsparse * t_iter, 1.5 * wsparse * t_iter


# ---------------------------------------------------------------- measured constants
@dataclass
class Measured:
    """Per-GPU snapshot bandwidths measured by bench.py on B200 (bytes/s).

    host: a record delivered to pinned host memory through the C ABI (`e2e`),
      the analogue of the reference's `pcie_bandwidth` (snapshots go to CPU
      memory first);
    device: the on-device snapshot + replicate rate per GPU (`value` / N),
      the budget when replicas stay in HBM of peers (NVLink);
    """
    host: float
    device: float
    source: str = ""

    @classmethod
    def from_bench(cls, line: str | dict) -> "Measured":
        j = json.loads(line) if isinstance(line, str) else line
        if j.get("unit") != "GB/s":
            raise ValueError("bench line: expected GB/s")
        n = max(1, int(j.get("n_gpus", 1)))
        return cls(host=float(j["e2e"]["value"]) * 1e9, device=float(j["value"]) / n * 1e9,
                   source=f"bench.py N={n}: e2e {j['e2e']['value']:.1f} GB/s, {j['value'] / n:.1f} GB/s/GPU")


def deepseek_layer_ops(layers: int = 1, experts: int = 64, expert_params: int = 7_898_100,
                       nonexpert_params: int = 80_140_000, gate_params: int = 100_000,
                       popularity=None) -> list[Operator]:
    """Layer-major operator ids of configs/deepseek_moe.json (core.hpp:105-134):
    E experts, then the non-expert block, then the gate, per layer."""
    ops = []
    for layer in range(layers):
        for e in range(experts):
            h = popularity[layer * experts + e] if popularity is not None else 0.0
            ops.append(Operator(len(ops), EXPERT, expert_params, hard=h))
        ops.append(Operator(len(ops), NON_EXPERT, nonexpert_params))
        ops.append(Operator(len(ops), GATE, gate_params))
    return ops


def compare(ops: list[Operator], plan: Precision, t_iter: float, reference_bandwidth: float, measured: Measured,
            ordering: int = HARD) -> dict:
    """The window the reference's constant gives against the windows the
    measured B200 constants give, with the recovery-time bounds of each."""
    out = {}
    for name, bw in (("reference_pcie", reference_bandwidth), ("b200_host", measured.host),
                     ("b200_device", measured.device)):
        s = build_schedule(ops, plan, bw, t_iter, ordering)
        lo, hi, exp = recovery_time_bounds_sparse(s.wsparse, t_iter)
        out[name] = {"bandwidth_gbs": bw / 1e9, "wsparse": s.wsparse, "o_active": s.o_active,
                     "fits_budget": s.fits_budget, "max_slot_gb": s.max_slot_bytes(ops, plan) / 1e9,
                     "recovery_s_max": hi, "recovery_s_expected": exp}
    out["source"] = measured.source
    return out


def iteration_time(t_stage: list[float], microbatches: int, t_sync: float, t_update: float) -> float:
    """GPipe-style iteration time (sim.hpp:35-47)."""
    return (microbatches + len(t_stage) - 1) * max(t_stage) + t_sync + t_update


def _main():
    import argparse
    ap = argparse.ArgumentParser(description="W and recovery bounds of configs/deepseek_moe.json under the "
                                             "reference's PCIe constant and the measured B200 constants")
    ap.add_argument("bench_json", help="file holding a bench.py JSON line")
    args = ap.parse_args()
    with open(args.bench_json) as f:
        line = [ln for ln in f.read().splitlines() if ln.strip().startswith("{")][-1]
    m = Measured.from_bench(line)
    # configs/deepseek_moe.json: 28 layers x (64 experts + NE + gate); profile
    # 12 stages x 0.12 s, 16 micro-batches, t_sync 0.1405, t_update 0.074
    t_iter = iteration_time([0.12] * 12, 16, 0.1405, 0.074)
    # popularity skew 0.5 (workload.skew): expert e of a layer gets (e + 1) ** -0.5
    pop = [(e % 64 + 1) ** -0.5 for e in range(28 * 64)]
    res = compare(deepseek_layer_ops(28, popularity=pop), Precision(), t_iter, 18.95e9, m)
    res["t_iter_s"] = t_iter
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    _main()
