#!/usr/bin/env python
"""Benchmark of the B200 checkpoint data path (BASELINE.json metric:
"snapshot+replicate GB/s/GPU and sparse-to-dense conversion time vs
HBM/NVLink roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload auto|deepseek|mixtral]

--gpus N > 1 without torchrun: the script relaunches itself under
torch.distributed.run (N ranks, one per GPU, 127.0.0.1); under torchrun the
world size must equal N.

A step = one training iteration's sparse snapshot: serialize_record(
take_sparse_snapshot(state, slot[i mod W])) packed on the GPU into the
byte-exact MLCK record (+ FNV-1a-64 trailer) and pushed to its replicas.
  workload auto = deepseek at N = 1, mixtral at N > 1:
  deepseek: "deepseek_moe_layer" (BASELINE configs[1]): one layer of
            proj/configs/deepseek_moe.json (64 x 7,898,100 + NE 80,140,000 +
            G 100,000 params), W=6, O=11, fp16 compute; replica = a second
            HBM buffer written by the same kernel.
  mixtral:  "mixtral_8x7b_ep" (configs[2]): 16 experts x 176,160,768 params
            per GPU (expert-parallel, weak scaling), W=4, O=4; each GPU pushes
            its record to r = min(2, N-1) ring peers over NVLink (CUDA IPC
            buffers; at N = 1 the replica is a second HBM buffer).  The N = 1
            line also carries this workload (`same_workload_n1`), so the
            1 -> N curve exists on one workload.
Then the sparse-to-dense conversion of one full window (configs[3]) with
fused Adam replay from logged gradients, localized recovery, the upstream
log (configs[4]), gradient-log capture and snapshot-beside-training
interference are timed on the same device.  `value` is the whole-job
aggregate (record bytes of all ranks / max-over-ranks time, the bench
contract); `per_gpu_gbs` is the metric's GB/s/GPU.  Rank 0 prints one JSON
line.  `--impl reference` times the reference's own CPU path (oracle/_ref:
the unmodified proj/include headers) on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

GB = 1e9
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------
def deepseek_layer():
    experts, p_e, p_ne, p_g = 64, 7_898_100, 80_140_000, 100_000
    pcs = [p_e] * experts + [p_ne, p_g]
    # order_operators(HardCount) with zero popularity: experts by id, NE, G
    ordered = list(range(experts)) + [experts, experts + 1]
    return dict(name="deepseek_moe_layer", param_counts=pcs, ordered=ordered, W=6, O=11, cb=2)


def mixtral_ep():
    experts, p_e = 16, 176_160_768  # d=4096, d_ff=14336, SwiGLU: 3*4096*14336
    return dict(name="mixtral_8x7b_ep", param_counts=[p_e] * experts, ordered=list(range(experts)), W=4, O=4,
                cb=2)


def schedule(wl):
    """generate_schedule (schedule.hpp:153-172)."""
    o, n = wl["ordered"], len(wl["ordered"])
    return [(o[k * wl["O"]:min((k + 1) * wl["O"], n)], o[min((k + 1) * wl["O"], n):]) for k in range(wl["W"])]


def record_bytes(wl, slot):
    pcs, cb = wl["param_counts"], wl["cb"]
    a, c = slot
    return 45 + 8 + sum(13 + 8 + 12 * pcs[i] for i in a) + sum(13 + cb * pcs[i] for i in c)


def payload_bytes(wl, slot):
    pcs, cb = wl["param_counts"], wl["cb"]
    a, c = slot
    return sum(12 * pcs[i] for i in a) + sum(cb * pcs[i] for i in c)


def meta_bytes(slot):
    n = len(slot[0]) + len(slot[1])
    segs = 2 * n + 1
    return 4 * n + 24 * segs + 45 + 13 * n + 8 * len(slot[0])


# --------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# --------------------------------------------------------------------------
class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    polled every 2 ms in a thread (a 12-step region is ~17 ms), else
    nvidia-smi every 20 ms; __enter__ returns once the sampler is live, so the
    samples cover the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits in the order of FIELDS[3:]
    NVML_BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None
        self.t_start = self.t_end = None
        self.stop = threading.Event()
        self.t = None
        self.source = None

    def _nvml_loop(self, nv, h):
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                break
            flags = ["Active" if r & b else "Not Active" for b in self.NVML_BITS]
            self.samples.append((time.monotonic(), [str(sm), str(mx), hex(r)] + flags))
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.t.start()
            self.source = "nvml, 2 ms"
        except Exception:
            self.t = None
        if self.t is None:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                     "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
                self.source = "nvidia-smi, 20 ms"
            except OSError:
                self.proc = None
        deadline = time.monotonic() + 10
        while self.t is not None and not self.samples and time.monotonic() < deadline:
            time.sleep(0.001)
        self.t_start = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.monotonic(), parts))

    def __exit__(self, *a):
        self.t_end = time.monotonic()
        if self.t is not None:
            # one more sample after the region ends (a region can be shorter than the period)
            n = len(self.samples)
            deadline = time.monotonic() + 0.2
            while len(self.samples) == n and time.monotonic() < deadline:
                time.sleep(0.001)
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        inside = [p for t, p in self.samples if self.t_start is not None and self.t_start <= t <= (self.t_end or t) + 0.05]
        if not inside and self.samples:
            inside = [self.samples[-1][1]]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "source": self.source}


def peaks():
    try:
        with open(PEAKS_PATH) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_pipes(kernel):
    """The compute-side bound of `kernel` from the same committed capture:
    issue-slot and ALU/FMA/tensor pipe utilisation (% of peak while active)."""
    pdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    try:
        names = sorted(n for n in os.listdir(pdir) if n.endswith("_ncu_summary.json"))
        with open(os.path.join(pdir, names[-1])) as fh:
            k = json.load(fh)["full_captures"][kernel]
        f = lambda key: float(k[key][0] if isinstance(k[key], list) else k[key])  # noqa: E731
        return {"issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "alu_pipe_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                "fma_pipe_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                "tensor_pipe_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                "source": f"profiles/{names[-1]}"}
    except (OSError, IndexError, KeyError, ValueError):
        return None


def ncu_traffic(kernel):
    """dram read+write bytes of one launch of `kernel` from the newest committed
    `ncu --set full` summary (profiles/rNN_ncu_summary.json, scripts/profile.sh)."""
    pdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    try:
        names = sorted(n for n in os.listdir(pdir) if n.endswith("_ncu_summary.json"))
        with open(os.path.join(pdir, names[-1])) as fh:
            s = json.load(fh)
        return float(s["full_captures"][kernel]["traffic_bytes"]), f"profiles/{names[-1]} (one launch)"
    except (OSError, IndexError, KeyError, ValueError):
        return None, None


# --------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Dist:
    def __init__(self, world, rank, local):
        self.world, self.rank, self.local = world, rank, local
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist, self.torch = dist, torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t)
        return float(t.item())

    def all_gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# --------------------------------------------------------------------------
# CPU leg (reference compiled from /root/reference; oracle/_ref)
# --------------------------------------------------------------------------
def cpu_pack_sample(wl, threads, iters=1):
    """The reference's take_sparse_snapshot + serialize_record on the host,
    `threads` independent shards of a bounded sample of slot 0."""
    import ctypes as C
    from oracle.oracle import load_reference
    ref = load_reference()
    if ref is None:
        return None
    pcs = wl["param_counts"]
    a, c = schedule(wl)[0]
    # per thread: one Full expert + CO experts in the slot's ratio (bounded)
    n_full, full_p = 1, pcs[a[0]]
    ratio = max(1, round(len(c) / max(1, len(a))))
    n_co, co_p = min(ratio, 5), pcs[c[0]] if c else 0
    if wl["name"] == "mixtral_8x7b_ep":  # 176M-param experts: scale the sample
        full_p, co_p = full_p // 16, co_p // 16
    blob = C.c_uint64()
    secs = C.c_double()
    bps = ref.lib.mlr_time_pack(threads, n_full, full_p, n_co, co_p, wl["cb"], iters, C.byref(blob), C.byref(secs))
    return dict(bytes_per_s=bps, seconds=secs.value, blob=blob.value, n_full=n_full, full_params=full_p, n_co=n_co,
                co_params=co_p, threads=threads, iters=iters)


def cpu_convert_sample(threads, scale=256):
    """The reference's sparse_to_dense_convert (recovery.hpp:180-227, its
    recompute replay included) and the merge + logged-gradient replay, on the
    configs[3] window shape scaled down by `scale` (64 experts + NE + G,
    W=6, O=11), `threads` independent engines."""
    import ctypes as C
    from oracle.oracle import load_reference
    ref = load_reference()
    if ref is None:
        return None
    L = ref.lib
    L.mlr_time_convert.restype = C.c_double
    L.mlr_time_convert.argtypes = [C.c_uint32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_uint32, C.c_uint32,
                                   C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    secs = (C.c_double * 2)()
    blob = C.c_uint64()
    steps = L.mlr_time_convert(threads, 64, 7_898_100 // scale, 80_140_000 // scale, 100_000 // scale, 6, 11, secs,
                               C.byref(blob))
    full_steps = 1_888_904_900  # configs[3]
    conv_rate = threads * steps / secs[0]
    replay_rate = threads * steps / secs[1]
    return {"threads": threads, "sample": f"configs[3] window shape / {scale} (64 x {7_898_100 // scale} + "
                                          f"{80_140_000 // scale} + {100_000 // scale} params, W=6, O=11), "
                                          f"{threads} independent engines",
            "element_steps_per_thread": steps, "convert_s": secs[0], "replay_s": secs[1],
            "convert_msteps_per_s": conv_rate / 1e6, "replay_msteps_per_s": replay_rate / 1e6,
            "convert_ms_extrapolated_configs3": 1000 * full_steps / conv_rate,
            "replay_ms_extrapolated_configs3": 1000 * full_steps / replay_rate}


def cpu_fnv_sample(mb=256):
    """The reference's fnv1a64 (digest.hpp:18-25) on one core over `mb` MiB:
    the byte-serial trailer of serialize_record and the check of parse_record."""
    import ctypes as C
    import numpy as np
    from oracle.oracle import load_reference
    ref = load_reference()
    if ref is None:
        return None
    L = ref.lib
    L.mlr_fnv1a64.restype = C.c_uint64
    L.mlr_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
    buf = np.random.default_rng(7).integers(0, 256, mb << 20, dtype=np.uint8)
    L.mlr_fnv1a64(buf.ctypes.data, 1 << 20, 0xCBF29CE484222325)  # warm
    t0 = time.perf_counter()
    L.mlr_fnv1a64(buf.ctypes.data, buf.size, 0xCBF29CE484222325)
    sec = time.perf_counter() - t0
    return {"threads": 1, "bytes": int(buf.size), "seconds": sec, "gbs": buf.size / sec / GB,
            "note": "byte-serial: one core is the reference's rate for any one record (no parallel FNV)"}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline_full(wl):
    """cpu_baseline: the headline all-core pack number plus the 1-core and
    all-core pack and conversion numbers of the reference."""
    n = cpu_threads()
    p_all = cpu_pack_sample(wl, n)
    if p_all is None:
        return None
    p_one = cpu_pack_sample(wl, 1)
    c_one = cpu_convert_sample(1)
    c_all = cpu_convert_sample(n)
    out = {"value": p_all["bytes_per_s"] / GB, "unit": "GB/s", "cores": n, "kind": "reference",
           "sample": (f"reference take_sparse_snapshot+serialize_record, per thread {p_all['n_full']} Full x "
                      f"{p_all['full_params']} + {p_all['n_co']} CO x {p_all['co_params']} params, "
                      f"{n} independent engines, {p_all['seconds']:.1f} s"),
           "pack_1core_gbs": p_one["bytes_per_s"] / GB, "pack_all_cores_gbs": p_all["bytes_per_s"] / GB,
           "conversion_1core": c_one, "conversion_all_cores": c_all, "fnv1a64_1core": cpu_fnv_sample()}
    out.update(host_info())
    return out


def AUTO_TRANSPORT(world):
    """What replica mode -1 (auto) picks: 2 (fused) for local replicas (N=1), 1 for peers."""
    return 2 if world == 1 else 1


METRIC = "snapshot+replicate GB/s/GPU and sparse-to-dense conversion time vs HBM/NVLink roofline"


def arm_config(wl, world):
    """The workload description both arms print (same metric, same config)."""
    slots = schedule(wl)
    r = 1 if world == 1 else min(2, world - 1)
    return {"workload": wl["name"], "params_per_gpu": sum(wl["param_counts"]), "wsparse": wl["W"],
            "o_active": wl["O"], "compute_bytes": wl["cb"], "replicas": r,
            "replica_target": "second HBM buffer" if world == 1 else "ring peers over NVLink (IPC)",
            "record_bytes_per_slot": [record_bytes(wl, sl) for sl in slots], "parallelism": f"ep{world}",
            "l2": "inputs larger than L2 (records 1.3-12.7 GB)"}


def cpu_threads():
    n = os.cpu_count() or 1
    return max(1, min(n, 32))


def pick_workload(args, world):
    name = args.workload if args.workload != "auto" else ("deepseek" if world == 1 else "mixtral")
    return deepseek_layer() if name == "deepseek" else mixtral_ep()


def run_reference(args, d: Dist):
    if d.rank != 0:
        return
    wl = pick_workload(args, d.world)
    threads = cpu_threads()
    vals, secs = [], 0.0
    for _ in range(args.warmup):
        cpu_pack_sample(wl, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = cpu_pack_sample(wl, threads)
        if s is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference tree absent)"}))
            return
        vals.append(s["bytes_per_s"] / GB)
        secs += s["seconds"]
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    sample = (f"per thread: {s['n_full']} Full x {s['full_params']} params + {s['n_co']} ComputeOnly x "
              f"{s['co_params']} params (slot-0 mix), {threads} independent engines")
    out = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "GB/s", "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * secs / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 (byte-exact container) / f32 Adam", "data": "synthetic",
        "config": arm_config(wl, d.world),
        "reference_path": "take_sparse_snapshot + serialize_record (snapshot.hpp:115-144, 204-241) compiled from "
                          f"/root/reference (oracle/_ref), {threads} host threads, bounded sample per step",
        "cpu_baseline": dict({"value": value, "unit": "GB/s", "cores": threads, "kind": "reference",
                              "sample": sample}, **host_info()),
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    if not args.no_convert:  # the conversion half of the metric on the same host cores
        out["conversion"] = cpu_convert_sample(threads)
    print(json.dumps(out))


# --------------------------------------------------------------------------
# upstream logging (configs[4]): one interior pipeline stage per GPU
# --------------------------------------------------------------------------
def bench_logging(ctx, d, mlck, iterations=3):
    """configs[4]: dp=2 x pp=4, M=8 micro-batches, boundary tensors
    [4096 tokens x 2048] fp32 = 33,554,432 B.  An interior stage owns 16
    entries per iteration (8 fwd sends + 8 bwd sends, engine.hpp:381-387,
    404-411) = 537 MB per GPU per iteration.  Each rank logs them (a) to a
    pinned host ring (kind 0, the paper's design: PCIe/C2C) and (b) to device
    HBM: its ring successor's buffer over NVLink (kind 2, CUDA IPC) at N > 1,
    a local ring at N = 1.  Copies run on the log's low-priority side stream;
    `overlap` is the slowdown of a concurrent HBM-bound kernel on the
    producer stream."""
    entry_floats, m, per_it = 4096 * 2048, 8, 16
    entry_b = 4 * entry_floats
    it_bytes = per_it * entry_b
    src = [ctx.alloc(entry_b) for _ in range(2)]  # the stage's send buffers
    for p in src:
        ctx.memset(p, 0x3c, entry_b)
    cap = 2 * it_bytes + (1 << 20)

    def run(log):
        log.sync()
        log.gc(1 << 62)  # empty ring
        t0 = time.perf_counter()
        for it in range(iterations):
            for mb in range(m):
                log.put(1000 + it, mb, 1, 0, src[mb & 1], entry_floats)       # fwd: boundary 1 (sender)
                log.put(1000 + it, mb, 1, 1, src[(mb + 1) & 1], entry_floats)  # bwd: boundary 1 (receiver side)
            log.sync()
            log.gc(1000 + it)  # keep one iteration (persisted window advanced)
        return (time.perf_counter() - t0) / iterations

    out = {"workload": "dp2 x pp4, M=8, [4096x2048] f32 boundary tensors (configs[4]); interior stage",
           "entries_per_iteration": per_it, "bytes_per_iteration": it_bytes}
    # raw copy-engine peaks for the same bytes (the roofline of a copy)
    hbuf = ctx.alloc_pinned(entry_b)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(per_it):
        ctx.d2h(hbuf, src[0], entry_b)
    ctx.synchronize()
    d2h_peak = it_bytes / (time.perf_counter() - t0) / GB
    ctx.free_pinned(hbuf)
    host = mlck.UpstreamLog(ctx, cap, kind=0)
    run(host)
    s = d.max(run(host))
    out["pinned_host"] = {"ms_per_iteration": 1000 * s, "gbs": it_bytes / s / GB,
                          "peak_gbs": d2h_peak, "peak_kind": "measured cudaMemcpyAsync D2H, same bytes",
                          "frac": it_bytes / s / GB / d2h_peak}
    host.close()
    # device ring: successor's HBM (IPC) at N > 1, local HBM at N = 1
    ring = ctx.alloc(cap)
    handles = d.all_gather(ctx.ipc_export(ring))
    opened = None
    if d.world > 1:
        opened = ctx.ipc_open(handles[(d.rank + 1) % d.world])
        dev = mlck.UpstreamLog(ctx, cap, kind=2, external=opened)
        target, peak, peak_kind = "successor HBM over NVLink (CUDA IPC, copy engine)", 782.0, "measured peer copy (scripts/micro/push.cu)"
    else:
        dev = mlck.UpstreamLog(ctx, cap, kind=2, external=ring)
        target, peak, peak_kind = ("local HBM ring (copy engine)", peaks()[0] / 2,
                                   "MEASURED_PEAKS hbm_gbs / 2 (a copy reads and writes every byte)")
    d.barrier()
    run(dev)
    d.barrier()
    s = d.max(run(dev))
    g = it_bytes / s / GB
    out["device_ring"] = {"target": target, "ms_per_iteration": 1000 * s, "gbs": g, "peak_gbs": peak,
                          "peak_kind": peak_kind, "frac": g / peak if peak else None}
    # overlap: an HBM-bound kernel on the producer stream with and without
    # the host-ring copies of one iteration running beside it
    n = 1 << 28
    a = ctx.alloc(8 * n)
    ctx.memset(a, 0, 8 * n)
    ctx.synchronize()

    def busy(reps):  # quantize_inplace-shaped HBM stream (read 4n, write 4n bytes)
        ctx.event_record(4)
        for _ in range(reps):
            ctx.quantize(a, a + 4 * n, n, 2)
        ctx.event_record(5)

    busy(2)
    ctx.synchronize()
    busy(16)
    ctx.synchronize()
    base_ms = ctx.event_ms(4, 5)
    host = mlck.UpstreamLog(ctx, cap, kind=0)
    host.set_async(True)  # the producer does not wait for the copies (it does not reuse src here)
    for mb in range(m):
        host.put(2000, mb, 1, 0, src[mb & 1], entry_floats)
        host.put(2000, mb, 1, 1, src[(mb + 1) & 1], entry_floats)
    busy(16)
    ctx.synchronize()
    host.sync()
    with_ms = ctx.event_ms(4, 5)
    host.close()
    out["overlap"] = {"producer": "quantize kernel stream, 16 x 2 GiB HBM (log in async mode)", "producer_kernel_ms": base_ms,
                      "with_host_logging_ms": with_ms, "slowdown": with_ms / base_ms - 1}
    dev.close()
    if opened:
        ctx.ipc_close(opened)
    d.barrier()
    for p in src + [ring, a]:
        ctx.free(p)
    return out


# --------------------------------------------------------------------------
# gradient-log capture (the replay's input)
# --------------------------------------------------------------------------
def bench_gradlog_capture(ctx, mlck, wl, st, iterations=4):
    """Per-iteration cost of logging the weight gradients the conversion
    replays: (a) copy capture -- the trainer's gradient buffers (here the
    state's m arrays stand in) copied into the log slot of the iteration on
    the ctx stream; (b) zero copy -- the trainer's backward writes straight
    into mlck_gradlog_slot, no extra traffic.  Plus the HBM the log holds."""
    pcs, W = wl["param_counts"], wl["W"]
    g = mlck.GradLog(ctx, pcs, W)
    srcs = [st.op_ptrs(i)[1] for i in range(len(pcs))]

    def capture(it):
        for i in range(len(pcs)):
            g.capture(it, i, srcs[i])

    capture(1)
    ctx.synchronize()
    ctx.event_record(6)
    for it in range(2, 2 + iterations):
        capture(it)
    ctx.event_record(7)
    ctx.synchronize()
    ms = ctx.event_ms(6, 7) / iterations
    it_bytes = 4 * sum(pcs)
    full_slot = {i: k for k, (a, _) in enumerate(schedule(wl)) for i in a}
    need = sum(4 * pcs[i] * (W - full_slot[i]) for i in range(len(pcs)))
    out = {"workload": wl["name"], "gradient_bytes_per_iteration": it_bytes,
           "copy_capture": {"ms_per_iteration": ms, "gbs": 2 * it_bytes / (ms / 1000) / GB,
                            "note": "D2D copy of every operator's gradient into the log (read + write)"},
           "zero_copy_capture": {"ms_per_iteration": 0.0,
                                 "note": "backward writes into mlck_gradlog_slot(iteration, op): no copy"},
           "hbm_resident_gb": g.nbytes / GB,
           "hbm_minimum_gb": need / GB,
           "resident_note": f"a ring of W={W} iterations x all operators; the replay reads only sum 4P(W-k) "
                            "(each operator's gradients after its Full slot)"}
    g.close()
    return out


# --------------------------------------------------------------------------
# snapshot beside training (snapshots overlap compute)
# --------------------------------------------------------------------------
def bench_interference(ctx, mlck, st, blobs, slots, dev, gemms=200):
    """A training-like stream (bf16 GEMMs 8192^3 on the tensor cores plus an
    HBM-bound elementwise pass per GEMM) on a high-priority stream, alone and
    with one snapshot (pack + hash + replica of slot 0) issued beside it.
    Reports the training slowdown and the snapshot's latency per setting."""
    import torch
    torch.cuda.set_device(dev)
    hi = torch.cuda.Stream(device=dev, priority=-1)
    lo = torch.cuda.Stream(device=dev, priority=0)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    x = torch.empty(1 << 28, device=dev, dtype=torch.float32)  # 1 GiB: the HBM-bound pass
    x.fill_(1.0)

    def train():
        with torch.cuda.stream(hi):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(gemms):
                torch.matmul(a, b, out=c)
                x.mul_(1.0000001)
            e1.record()
        return e0, e1

    def run(stream_handle, reserve, with_snapshot):
        ctx.set_stream(stream_handle)
        ctx.set_hash_reserve(reserve)
        torch.cuda.synchronize()
        e0, e1 = train()
        if with_snapshot:
            ctx.event_record(8)
            a0, c0 = slots[0]
            mlck.snapshot_record(st, a0, c0, 0, 1, 1000, len(slots), blobs[0])
            ctx.event_record(9)
        torch.cuda.synchronize()
        ctx.synchronize()
        t = e0.elapsed_time(e1)
        snap = ctx.event_ms(8, 9) if with_snapshot else None
        return t, snap

    run(None, 0, False)
    base = statistics.median(run(None, 0, False)[0] for _ in range(3))
    out = {"training": f"{gemms} x (bf16 GEMM 8192^3 + 1 GiB fp32 elementwise), high-priority stream",
           "training_ms_alone": base, "settings": {}}
    for name, handle, reserve in (("ctx stream (highest priority), all SMs", None, 0),
                                  ("low-priority stream, all SMs", lo.cuda_stream, 0),
                                  ("low-priority stream, hash on 74 SMs", lo.cuda_stream, 74)):
        run(handle, reserve, True)
        res = [run(handle, reserve, True) for _ in range(3)]
        t = statistics.median(r[0] for r in res)
        sn = statistics.median(r[1] for r in res)
        out["settings"][name] = {"training_ms": t, "slowdown": t / base - 1, "delay_ms": t - base, "snapshot_ms": sn}
    ctx.set_stream(None)
    ctx.set_hash_reserve(0)
    best = min(out["settings"].values(), key=lambda v: v["slowdown"])
    out["best_slowdown"] = best["slowdown"]
    # the same delay against a real iteration: DeepSeek-MoE's t_iter in the
    # reference's profile (sim.hpp:35-47, PAPER.md) is 3.45 s
    out["best_delay_vs_deepseek_iteration"] = best["delay_ms"] / 3450.0
    del a, b, c, x
    torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------------
# GPU leg
# --------------------------------------------------------------------------
def bench_snapshot_n1(ctx, mlck, wl, args):
    """Snapshot steps of `wl` on one GPU: one record buffer + a replica in a
    second HBM buffer (auto transport: the fused kernel), records rotating through the slots."""
    pcs, cb, W = wl["param_counts"], wl["cb"], wl["W"]
    slots = schedule(wl)
    sizes = [record_bytes(wl, sl) for sl in slots]
    cap = max(sizes)
    st = mlck.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=7, step=10)
    st.set_meta(1000, 7)
    blob = mlck.Blob(ctx, cap)
    rep = ctx.alloc(cap)
    blob.add_replica(rep, cap)

    def step(i):
        a, c = slots[i % W]
        mlck.snapshot_record(st, a, c, i % W, 1, 1000, W, blob)

    for i in range(args.warmup):
        step(i)
    ctx.synchronize()
    ctx.event_record(0)
    for i in range(args.steps):
        step(i)
    ctx.event_record(1)
    ctx.synchronize()
    ms = ctx.event_ms(0, 1)
    total = sum(sizes[i % W] for i in range(args.steps))
    out = {"workload": wl["name"], "n_gpus": 1, "replica_target": "second HBM buffer (auto transport 2, fused)",
           "ms_per_step": ms / args.steps, "value": total / (ms / 1000) / GB, "unit": "GB/s",
           "record_bytes_per_slot": sizes}
    st.close()
    blob.close()
    ctx.free(rep)
    return out


def run_ours(args, d: Dist):
    from paper_2412_15411_b200 import mlck

    dev = d.local
    ctx = mlck.Context(dev)
    ctx.set_hash_async(bool(args.hash_async))
    ctx.set_hash_reserve(args.hash_reserve)
    ctx.set_convert_overlap(args.convert_overlap)
    if args.replica_mode != -1:
        ctx.set_replica_mode(args.replica_mode)
    wl = pick_workload(args, d.world)
    pcs, cb, W = wl["param_counts"], wl["cb"], wl["W"]
    slots = schedule(wl)
    sizes = [record_bytes(wl, s) for s in slots]
    cap = max(sizes)
    r = 1 if d.world == 1 else min(2, d.world - 1)

    st = mlck.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=7 + d.rank, step=10)
    st.set_meta(1000, 7)

    # record buffers: one per slot (the conversion needs the whole window)
    blobs = [mlck.Blob(ctx, cap) for _ in range(W)]
    recv, opened = [], []
    if d.world == 1:
        rep = [ctx.alloc(cap) for _ in range(W)]
        for b, p in zip(blobs, rep):
            b.add_replica(p, cap)
        recv = rep
    else:
        # each GPU hosts r receive buffers, one per ring predecessor; the
        # pack kernel writes the peers' buffers directly (NVLink stores)
        from paper_2412_15411_b200 import placement
        recv = [ctx.alloc(cap) for _ in range(r)]
        targets = placement.exchange_handles(d.all_gather, [ctx.ipc_export(p) for p in recv], d.rank,
                                             d.world)
        for handle, _peer in targets:
            ptr = ctx.ipc_open(handle)
            opened.append(ptr)
            for b in blobs:
                b.add_replica(ptr, cap)

    def step(i):
        k = i % W
        a, c = slots[k]
        mlck.snapshot_record(st, a, c, k, 1, 1000, W, blobs[k])

    for i in range(args.warmup):
        step(i)
    ctx.synchronize()

    # ---- timed region (device events, barrier + sync both sides).  The
    # clock sampler starts first (it takes a variable time to deliver its
    # first sample), so the barrier lines the ranks up on the region itself.
    with ClockSampler(dev) as clk:
        d.barrier()
        ctx.synchronize()
        launches0 = ctx.kernel_launches
        ctx.event_record(0)
        for i in range(args.steps):
            step(i)
        ctx.event_record(1)
        launches = ctx.kernel_launches - launches0  # our kernels launched in the timed region
        ctx.synchronize()
        d.barrier()
    ms_local = ctx.event_ms(0, 1)
    ms = d.max(ms_local)
    bytes_local = sum(sizes[i % W] for i in range(args.steps))
    total_bytes = d.sum(bytes_local)
    value = total_bytes / (ms / 1000) / GB
    transport = args.replica_mode if args.replica_mode != -1 else AUTO_TRANSPORT(d.world)  # the timed transport

    # ---- per-kernel breakdown (CUDA events around each launch) of the timed
    # configuration -- N=1, transport 2: one fused FNV kernel loads the
    # record's chunks from the state arena, hashes them and stores the record
    # and its local replica; N>1, transport 1: pack
    # kernel, then the copy engines push to the ring peers while the FNV
    # kernel hashes -- plus every other transport as a whole-step ablation.
    hbm_peak, peak_kind = peaks()
    payload = [payload_bytes(wl, slots[i % W]) for i in range(args.steps)]
    rec = [sizes[i % W] for i in range(args.steps)]
    local_rep = r if d.world == 1 else 0  # replicas written to local HBM
    ctx.set_timing(True)
    for i in range(args.steps):
        step(i)
    tim = ctx.timings()
    ctx.set_timing(False)

    def step_ms(mode):
        ctx.set_replica_mode(mode)
        for i in range(2):
            step(i)
        d.barrier()
        ctx.synchronize()
        ctx.event_record(0)
        for i in range(args.steps):
            step(i)
        ctx.event_record(1)
        ctx.synchronize()
        d.barrier()
        return d.max(ctx.event_ms(0, 1)) / args.steps

    names = {0: "pack kernel stores the replicas, then hash",
             1: "pack, then copy-engine push beside the hash",
             2: "one fused gather + store + hash kernel",
             3: "pack, then a push kernel on 16 reserved SMs beside the hash",
             4: "pack, hash, then copy-engine push (no overlap)",
             5: "pack, then the hash kernel stores the replicas"}
    ablations = {}
    for m in names:
        if m != transport:
            t = step_ms(m)
            ablations[f"transport {m}"] = {"ms_per_step": t, "value": total_bytes / (t * args.steps / 1000) / GB,
                                           "what": names[m]}
    ctx.set_replica_mode(args.replica_mode)
    pack_ms = [t for n, t in tim if n == "pack"]
    fnv_ms = [t for n, t in tim if n == "fnv"]
    push_ms = [t for n, t in tim if n == "push"]
    fused_ms = [t for n, t in tim if n == "pack_fnv"]

    def kstat(ms_list, total_bytes, note):
        return {"ms_avg": statistics.mean(ms_list), "launches": len(ms_list),
                "bytes_per_launch": total_bytes / len(ms_list),
                "gbs": total_bytes / (sum(ms_list) / 1000) / GB, "bytes": note}

    pack_note = "HBM: payload read + record write" + (f" + {local_rep} local replica write" if local_rep else "")
    kernels = {}
    if fused_ms:
        kernels["pack_fnv"] = kstat(fused_ms, sum(payload) + (1 + local_rep) * sum(rec),
                                    pack_note + " (one fnv_kernel<fused>: TMA loads from the sources, hash, "
                                                "TMA stores)")
    if pack_ms:
        kernels["pack"] = kstat(pack_ms, sum(payload) + (1 + local_rep) * sum(rec), pack_note)
    if fnv_ms:
        kernels["fnv"] = kstat(fnv_ms, sum(rec), "HBM: record read (ALU-bound 8-bit automaton)")
    if push_ms:
        kernels["push"] = kstat(push_ms, r * sum(rec), "replica copies on the copy engines beside the hash (NVLink egress)")
    kd = kernels["pack_fnv"] if fused_ms else kernels["fnv"]
    ach = kd["bytes_per_launch"] / (kd["ms_avg"] / 1000) / GB
    traffic, traffic_src = ncu_traffic("fnv_kernel")
    if d.world > 1 and traffic is not None:
        # the committed capture is an N=1 launch (config-2 record); N>1 hashes config-3 records
        traffic, traffic_src = None, f"none: {traffic_src} is an N=1 (config-2) launch, not this workload's"
    roofline = {"bound": "hbm", "kernel": "pack_fnv" if fused_ms else "fnv", "transport": transport, "achieved": ach,
                "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "peak_kind": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
                "per_launch_bytes": kd["bytes_per_launch"],
                "compute_side": ncu_pipes("fnv_kernel"),
                "note": ("the step's one kernel (fused: TMA loads from the sources, hash, TMA stores of the record and "
                         "its replica; achieved = payload read + record and replica writes per launch)" if fused_ms else
                         "dominant kernel of the step (the pack kernel alone: kernels['pack'])") +
                        "; bound by the integer ALU work of the FNV automaton and its per-round look-back latency, "
                        "not by HBM (compute_side: issue / pipe utilisation from the committed ncu capture; "
                        "DESIGN.md 3.2)"}
    if d.world > 1:
        nv_peak = 782.0  # one copy engine, GPU->peer (scripts/micro/push.cu on this pool)
        egress = r * bytes_local / (ms_local / 1000) / GB
        roofline_nvlink = {"bound": "nvlink", "achieved": egress, "peak": nv_peak, "unit": "GB/s",
                           "frac": egress / nv_peak, "peak_kind": "measured peer copy (scripts/micro/push.cu)"}
    else:
        roofline_nvlink = None

    # ---- e2e: the record delivered to pinned host memory through the C ABI
    hbuf = ctx.alloc_pinned(cap)
    scratch = blobs[0]
    e2e_steps = max(1, min(args.steps, 6))
    for i in range(min(2, e2e_steps)):
        a, c = slots[i % W]
        mlck.snapshot_record_host(st, a, c, i % W, 1, 1000, W, scratch, hbuf, cap)
    d.barrier()
    t0 = time.perf_counter()
    e2e_bytes = 0
    h2d = 0
    for i in range(e2e_steps):
        a, c = slots[i % W]
        e2e_bytes += mlck.snapshot_record_host(st, a, c, i % W, 1, 1000, W, scratch, hbuf, cap)
        h2d += meta_bytes(slots[i % W])
    e2e_s = d.max(time.perf_counter() - t0)
    e2e_val = d.sum(e2e_bytes) / e2e_s / GB
    ctx.free_pinned(hbuf)

    # ---- conversion of one full window with fused Adam replay (configs[3])
    conv = None
    if not args.no_convert:
        for k in range(W):  # the window's records, slot k taken at state a+k
            a, c = slots[k]
            mlck.snapshot_record(st, a, c, k, 1, 1000, W, blobs[k])
        g = mlck.GradLog(ctx, pcs, W)
        g.fill_synthetic(1001, W, seed=11 + d.rank)
        # the dense result overwrites the live arena (the snapshot phase is
        # over): at N >= 3 a second 39 GB arena does not fit beside the window
        out = st
        mlck.sparse_to_dense_convert(out, blobs, 1000, W, 7, g)  # warm-up
        ctx.synchronize()
        reps = max(1, min(5, args.steps))
        ctx.event_record(4)  # each conversion between its own events; the median is reported
        for i in range(reps):
            mlck.sparse_to_dense_convert(out, blobs, 1000, W, 7, g)
            ctx.event_record(5 + i)
        ctx.synchronize()
        conv_reps = [ctx.event_ms(4 + i, 5 + i) for i in range(reps)]
        conv_ms = d.max(statistics.median(conv_reps))
        ctx.set_timing(True)
        mlck.sparse_to_dense_convert(out, blobs, 1000, W, 7, g)
        ctim = ctx.timings()
        ctx.set_timing(False)
        # cold records (loaded from files or a peer: no witness) -- every
        # record hashed from scratch with the look-back kernel
        ctx.set_witness(False)
        mlck.sparse_to_dense_convert(out, blobs, 1000, W, 7, g)
        ctx.synchronize()
        ctx.event_record(2)
        for _ in range(reps):
            mlck.sparse_to_dense_convert(out, blobs, 1000, W, 7, g)
        ctx.event_record(3)
        ctx.synchronize()
        conv_cold_ms = d.max(ctx.event_ms(2, 3) / reps)
        ctx.set_witness(True)
        # recovery from the replicas (N=1: the local replica buffers) with their
        # witnesses sent along (mlck_blob_add_replica_witness), wrapped in place
        conv_rep_ms = None
        if d.world == 1:
            wcap = mlck.witness_bytes(cap)
            wit = [ctx.alloc(wcap) for _ in range(W)]
            for b, wp in zip(blobs, wit):
                b.add_replica_witness(wp, wcap)
            for k in range(W):
                a, c = slots[k]
                mlck.snapshot_record(st, a, c, k, 1, 1000, W, blobs[k])
            ctx.synchronize()
            views = [mlck.Blob.wrap(ctx, rep[k], blobs[k].size, wit[k]) for k in range(W)]
            mlck.sparse_to_dense_convert(out, views, 1000, W, 7, g)
            ctx.synchronize()
            ctx.event_record(2)
            for _ in range(reps):
                mlck.sparse_to_dense_convert(out, views, 1000, W, 7, g)
            ctx.event_record(3)
            ctx.synchronize()
            conv_rep_ms = ctx.event_ms(2, 3) / reps
            for v in views:
                v.close()
            for b in blobs:
                b.clear_replicas()
                b.add_replica(rep[blobs.index(b)], cap)
            for wp in wit:
                ctx.free(wp)
        full_slot = {i: k for k, (a, _) in enumerate(slots) for i in a}
        grads_b = sum(4 * pcs[i] * (W - full_slot[i]) for i in range(len(pcs)))
        dense_b = sum((12 + cb) * p for p in pcs)
        blobs_b = sum(sizes)
        alg = blobs_b + grads_b + dense_b
        steps_e = sum(pcs[i] * (W - full_slot[i]) for i in range(len(pcs)))
        per = {}
        for n, t in ctim:
            per.setdefault(n, []).append(t)
        replay_ms = sum(per.get("replay", [0.0]))
        replay_bytes = sum(12 * pcs[i] for i in range(len(pcs))) + grads_b + dense_b
        conv = {
            "workload": "deepseek_moe_layer window W=6 (configs[3])" if d.world == 1 else
                        f"{wl['name']} window W={W}",
            "ms": conv_ms, "ms_each_run": conv_reps, "ms_cold_records": conv_cold_ms,
            "ms_from_replicas_with_witness": conv_rep_ms,
            "verification": "records this context hashed are re-verified against their witness (exact, "
                            "DESIGN 3.2); ms_cold_records: no witness, every record hashed with the look-back "
                            "kernel (records from files / peers); ms_from_replicas_with_witness: the window "
                            "converted from blobs wrapped over its replica buffers, the witnesses sent along",
            "algorithmic_bytes": alg, "adam_element_steps": steps_e,
            "achieved_gbs": alg / (conv_ms / 1000) / GB, "frac_hbm": alg / (conv_ms / 1000) / GB / hbm_peak,
            "roofline_ms": alg / (hbm_peak * GB) * 1000,
            "kernels": {n: {"ms_total": sum(v), "launches": len(v)} for n, v in per.items()},
            "replay_kernel": {"ms": replay_ms, "bytes": replay_bytes,
                              "gbs": replay_bytes / (replay_ms / 1000) / GB if replay_ms else None},
        }
        g.close()
    # localized recovery (recovery.hpp:240-289): one failed
    # pipeline stage = a quarter of the operators, from the same window, plus 3
    # lost iterations after it (N = 1: at N >= 3 a W+3-iteration gradient log
    # of the 2.8 G-parameter shard does not fit beside the window)
    if conv is not None and d.world == 1:
        extra = 3
        g = mlck.GradLog(ctx, pcs, W + extra)
        g.fill_synthetic(1001, W + extra, seed=11 + d.rank)
        scope = list(range(len(pcs) // 4))
        target = 1000 + W + extra
        mlck.localized_recover(out, scope, blobs, 1000, W, 7, g, target)  # warm-up
        ctx.synchronize()
        ctx.event_record(2)
        for _ in range(reps):
            mlck.localized_recover(out, scope, blobs, 1000, W, 7, g, target)
        ctx.event_record(3)
        ctx.synchronize()
        loc_ms = d.max(ctx.event_ms(2, 3) / reps)
        ctx.set_timing(True)
        mlck.localized_recover(out, scope, blobs, 1000, W, 7, g, target)
        ltim = ctx.timings()
        ctx.set_timing(False)
        lper = {}
        for n, t in ltim:
            lper.setdefault(n, []).append(t)
        steps_l = {i: W + extra - full_slot[i] for i in scope}
        loc_bytes = blobs_b + sum(12 * pcs[i] + 4 * pcs[i] * steps_l[i] + (12 + cb) * pcs[i] for i in scope)
        conv["localized_recovery"] = {
            "workload": f"{len(scope)} of {len(pcs)} operators (one of 4 stages), window W={W} + {extra} lost "
                        "iterations (SURVEY 8(f)-1)",
            "ms": loc_ms, "algorithmic_bytes": loc_bytes, "achieved_gbs": loc_bytes / (loc_ms / 1000) / GB,
            "adam_element_steps": sum(pcs[i] * steps_l[i] for i in scope),
            "kernels": {n: {"ms_total": sum(v), "launches": len(v)} for n, v in lper.items()},
            "note": "every record of the window is verified (parse_checked) before use, as the reference does"}
        g.close()

    # ---- upstream logging (configs[4])
    logging = None if args.no_log else bench_logging(ctx, d, mlck)

    # ---- parity spot check on this run's bytes (trailer vs CPU oracle FNV)
    parity = None
    if d.rank == 0 and not args.no_parity:
        from oracle.oracle import Oracle
        orc = Oracle()
        k = 5 if W > 5 else W - 1
        host = blobs[k].to_host()
        parity = (int.from_bytes(host[-8:], "little") == orc.fnv1a64(np.frombuffer(host[:-8], dtype=np.uint8)))
        if d.world == 1:
            parity = parity and ctx.download(recv[k], len(host)) == host

    # ---- gradient-log capture and snapshot beside training (N = 1)
    extras = {}
    if d.world == 1 and not args.no_extras:
        extras["gradlog_capture"] = bench_gradlog_capture(ctx, mlck, wl, st)
        extras["interference"] = bench_interference(ctx, mlck, st, blobs, slots, dev)

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu:
        cpu = cpu_baseline_full(wl)

    # ---- the configs[2] workload at N = 1 (replica in a second HBM buffer),
    # so the 1 -> N scaling curve has a point on one workload
    if d.world == 1 and not args.no_extras and wl["name"] != "mixtral_8x7b_ep":
        st.close()
        for b in blobs:
            b.close()
        for p in recv:
            ctx.free(p)
        recv = []
        extras["same_workload_n1"] = bench_snapshot_n1(ctx, mlck, mixtral_ep(), args)

    clocks = clk.summary()
    launches_total = ctx.kernel_launches
    if d.rank == 0:
        res = {
            "metric": METRIC,
            "value": value, "unit": "GB/s", "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 (byte-exact container) / f32 Adam", "data": "synthetic",
            "config": arm_config(wl, d.world),
            "per_gpu_gbs": value / d.world,
            "roofline": roofline,
            "roofline_nvlink": roofline_nvlink,
            "kernels": kernels,
            "transport_ablations": ablations,
            "conversion": conv,
            "logging": logging,
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": h2d // e2e_steps,
                    "d2h_bytes_per_step": e2e_bytes // e2e_steps, "path": "mlck_snapshot_record_host -> pinned host"},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "gpu_launches_total_run": launches_total,
            "parity_trailer_ok": parity,
            "clocks": clocks,
        }
        res.update(extras)
        print(json.dumps(res))

    for p in opened:
        ctx.ipc_close(p)
    d.barrier()


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "deepseek", "mixtral"])
    ap.add_argument("--no-convert", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-log", action="store_true")
    ap.add_argument("--hash-async", type=int, default=0, help="trailer hash off the pack's critical path (1/0)")
    ap.add_argument("--convert-overlap", type=int, default=0, help="SMs verifying beside the conversion replay")
    ap.add_argument("--replica-mode", type=int, default=-1, help="snapshot transport (-1 auto, 0-6)")
    ap.add_argument("--hash-reserve", type=int, default=0, help="SMs the hash kernel leaves to the next pack")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the N=1 same-workload leg, gradient-log capture and interference keys")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch under torchrun (the driver's own launch sets WORLD_SIZE)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    d = Dist(world, rank, local)
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_ours(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
