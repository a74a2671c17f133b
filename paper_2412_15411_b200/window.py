"""Window lifecycle and durability of sparse checkpoints.

`SparseCheckpoint` mirrors the reference's struct (snapshot.hpp:300-335) over
device blobs: the W records of one window in slot order plus per-record
replication counters.  Here the counters are driven by the device: a record's
replicas count once its push has completed (mlck_blob_replication), and a
durable file copy counts as one more (`save`).

`WindowRing` is the policy of PAPER.md:206: "MoEtion always maintains one
persisted checkpoint and another in-flight, garbage-collecting the oldest
checkpoint after persisting a new one".  Records go to the in-flight window
whose range holds their iteration (capture_windows, verify.hpp:63-84: the
record after state s belongs to window floor(s / W) * W); a window becomes
the persisted one once it is complete and every record reached the
replication target, and the window it replaces is released (its blobs go back
to a pool for reuse, and `on_persist` gets the new window start -- the
caller's gc_logs point, engine.hpp:90-94).
"""
from __future__ import annotations

import json
import os

from . import mlck

_MANIFEST = "window.json"


class SparseCheckpoint:
    """W serialized records of one window plus replication bookkeeping."""

    def __init__(self, window_start: int, wsparse: int, replication_target: int = 2):
        if wsparse < 1:
            raise ValueError("wsparse must be >= 1")
        self.window_start = window_start
        self.wsparse = wsparse
        self.replication_target = replication_target
        self.blobs: list[mlck.Blob] = []
        self.replication: list[int] = []   # peer copies per record
        self.durable: list[int] = []       # file copies per record

    def add_record(self, blob: mlck.Blob):
        """snapshot.hpp:306-309; the blob holds the serialized record."""
        if self.complete():
            raise RuntimeError("sparse checkpoint window is full")
        self.blobs.append(blob)
        self.replication.append(0)
        self.durable.append(0)

    def complete(self) -> bool:
        return len(self.blobs) == self.wsparse

    def poll(self):
        """Refresh the counters from the device (non-blocking)."""
        for k, b in enumerate(self.blobs):
            self.replication[k] = max(self.replication[k], b.replication() + self.durable[k])

    def persisted(self) -> bool:
        """snapshot.hpp:313-318."""
        return self.complete() and all(r >= self.replication_target for r in self.replication)

    def check_coverage(self, op_count: int, compute_bytes: int):
        mlck.check_coverage(self.blobs, op_count, compute_bytes)

    def record_path(self, directory: str, k: int) -> str:
        return os.path.join(directory, f"window_{self.window_start}_slot_{k}.mlck")

    def save(self, directory: str) -> list[str]:
        """Persist every record (MLCK v1 bytes, the reference's blob format) and
        a manifest; each file counts as one more durable copy."""
        os.makedirs(directory, exist_ok=True)
        paths = []
        for k, b in enumerate(self.blobs):
            path = self.record_path(directory, k)
            b.save(path)
            self.durable[k] += 1
            paths.append(path)
        man = {"format": "MLCK", "version": 1, "window_start": self.window_start, "wsparse": self.wsparse,
               "records": [os.path.basename(p) for p in paths]}
        tmp = os.path.join(directory, _MANIFEST + ".tmp")
        with open(tmp, "w") as f:
            json.dump(man, f)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, os.path.join(directory, _MANIFEST))  # the manifest lands last, atomically
        self.poll()
        return paths

    @classmethod
    def load(cls, ctx: mlck.Context, directory: str, replication_target: int = 2) -> "SparseCheckpoint":
        """A saved window back in device blobs (records are verified by
        parse_record / the conversion, not here)."""
        with open(os.path.join(directory, _MANIFEST)) as f:
            man = json.load(f)
        if man.get("format") != "MLCK" or man.get("version") != 1:
            raise RuntimeError("persist: unsupported window manifest")
        ck = cls(man["window_start"], man["wsparse"], replication_target)
        for name in man["records"]:
            ck.add_record(mlck.Blob.load(ctx, os.path.join(directory, name)))
            ck.durable[-1] = 1
        ck.poll()
        return ck


class WindowRing:
    """One persisted window plus the in-flight ones."""

    def __init__(self, ctx: mlck.Context, wsparse: int, replication_target: int = 2, on_persist=None):
        self.ctx = ctx
        self.wsparse = wsparse
        self.replication_target = replication_target
        self.on_persist = on_persist
        self.persisted: SparseCheckpoint | None = None
        self.in_flight: list[SparseCheckpoint] = []
        self._free: list[mlck.Blob] = []

    def window_of(self, state_index: int) -> int:
        """capture_windows: the record after state s belongs to window floor(s / W) * W."""
        return state_index // self.wsparse * self.wsparse

    def acquire(self, capacity: int) -> mlck.Blob:
        """A blob for the next record: a released one (with its replica
        targets, whose old copies belong to the collected window) or a new one.
        Blobs grow on demand, so `capacity` is only a hint."""
        return self._free.pop() if self._free else mlck.Blob(self.ctx, capacity)

    def add_record(self, state_index: int, blob: mlck.Blob) -> SparseCheckpoint:
        ws = self.window_of(state_index)
        win = next((w for w in self.in_flight if w.window_start == ws), None)
        if win is None:
            if self.persisted is not None and ws <= self.persisted.window_start:
                raise RuntimeError(f"record for window {ws} is older than the persisted window "
                                   f"{self.persisted.window_start}")
            win = SparseCheckpoint(ws, self.wsparse, self.replication_target)
            self.in_flight.append(win)
            self.in_flight.sort(key=lambda w: w.window_start)
        win.add_record(blob)
        return win

    def _release(self, win: SparseCheckpoint):
        self._free.extend(win.blobs)
        win.blobs = []

    def poll(self) -> bool:
        """Refresh replication; promote the newest persisted in-flight window
        and garbage-collect the one it replaces (and any older in-flight).
        Returns True when a new window became the persisted one."""
        newest = None
        for w in self.in_flight:
            w.poll()
            if w.persisted():
                newest = w
        if newest is None:
            return False
        old = [self.persisted] if self.persisted is not None else []
        old += [w for w in self.in_flight if w.window_start < newest.window_start]
        self.in_flight = [w for w in self.in_flight if w.window_start > newest.window_start]
        self.persisted = newest
        for w in old:
            self._release(w)
        if self.on_persist:
            self.on_persist(newest.window_start)
        return True
