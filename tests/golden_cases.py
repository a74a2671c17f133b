"""Loaders for the committed golden vectors (tests/golden/, generated from the
real reference by tests/golden/make_golden.py).  Shared by the oracle tests
(CPU) and the GPU parity tests."""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest() -> dict:
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


def load_npz(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@dataclass
class GoldenCase:
    name: str
    meta: dict
    d: object  # NpzFile

    @property
    def W(self):
        return self.meta["W"]

    @property
    def T(self):
        return self.meta["T"]

    @property
    def n_ops(self):
        return self.meta["n_ops"]

    @property
    def compute_bytes(self):
        return int(self.meta["cfg"]["compute_bytes"])

    @property
    def data_seed(self):
        return int(self.meta["data_seed"])

    @property
    def optimizer(self):
        c = self.meta["cfg"]
        return dict(kind=int(c["optimizer_kind"]), lr=c["lr"], beta1=c["beta1"], beta2=c["beta2"], eps=c["eps"])

    def slot(self, k):
        a, c = self.meta["slots"][k]
        return list(a), list(c)

    def op(self, s, i):
        d = self.d
        return dict(master=d[f"s{s}_op{i}_master"], m=d[f"s{s}_op{i}_m"], v=d[f"s{s}_op{i}_v"],
                    compute=d[f"s{s}_op{i}_compute"], step=int(d[f"s{s}_op{i}_step"][0]))

    def grads(self, it, i):
        return self.d[f"g{it}_op{i}"]

    def blob(self, s) -> bytes:
        return self.d[f"s{s}_blob"].tobytes()

    def mlst(self, s) -> bytes:
        return self.d[f"s{s}_mlst"].tobytes()

    def window_blobs(self, w):
        return [self.blob(w + k) for k in range(self.W)]

    def converted(self, w) -> bytes:
        return self.d[f"conv_w{w}"].tobytes()

    def localized(self):
        """[(window, target, stage_lo, stage_hi)] with a reference result."""
        return [tuple(x) for x in self.meta.get("localized", [])]

    def scope(self, lo, hi):
        return [i for i, st in enumerate(self.meta["stage_of_op"]) if lo <= st <= hi]

    def localized_image(self, w, target, lo, hi):
        """Parsed scope image of localized_recover: (iteration, {id: (step, master, m, v)})."""
        b = self.d[f"loc_w{w}_t{target}_s{lo}_{hi}"].tobytes()
        it = int.from_bytes(b[0:8], "little")
        n = int.from_bytes(b[8:12], "little")
        pos, ops = 12, {}
        for _ in range(n):
            i = int.from_bytes(b[pos:pos + 4], "little")
            step = int.from_bytes(b[pos + 4:pos + 12], "little")
            P = int.from_bytes(b[pos + 12:pos + 20], "little")
            pos += 20
            arrs = [np.frombuffer(b, dtype=np.float32, count=P, offset=pos + 4 * P * j) for j in range(3)]
            pos += 12 * P
            ops[i] = (step, *arrs)
        assert pos == len(b)
        return it, ops

    def header(self, s):
        w = s // self.W * self.W
        return dict(kind=1, iteration=s, window_start=w, wsparse=self.W, slot=s % self.W,
                    data_seed=self.data_seed)

    def record_entries(self, s):
        """Entries of the slot (s mod W) record of state s, sorted by id
        (take_sparse_snapshot, snapshot.hpp:204-241)."""
        active, co = self.slot(s % self.W)
        ents = []
        for i in active:
            o = self.op(s, i)
            ents.append(dict(id=i, mode=0, param_count=o["master"].size, step=o["step"], master=o["master"],
                             m=o["m"], v=o["v"]))
        for i in co:
            o = self.op(s, i)
            ents.append(dict(id=i, mode=1, param_count=o["compute"].size, compute=o["compute"]))
        ents.sort(key=lambda e: e["id"])
        return ents

    def log_entries(self):
        keys = self.d["log_keys"]
        return [(tuple(int(x) for x in keys[j]), self.d[f"log_{j}"]) for j in range(keys.shape[0])]


CASE_NAMES = ["verify_toy", "six_op_cb1", "six_op_cb4", "toy_sgd", "w1", "dp2_pp2"]


def load_case(name: str) -> GoldenCase:
    return GoldenCase(name, manifest()["cases"][name], load_npz(name))
