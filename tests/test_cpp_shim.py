"""The C++ drop-in (include/moelab_b200/checkpoint.hpp over the C ABI) run
the way the reference's harness runs moelab: a W-record window captured from
the golden states of the real reference, coverage, conversion -- byte-equal
to the reference's records and converted dense state."""
import os
import struct
import subprocess

import numpy as np
import pytest

from golden_cases import load_case
from oracle.oracle import ref_conversion_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "shim_parity")


def write_case(c, w, path):
    opt = c.optimizer
    out = bytearray()
    out += struct.pack("<IIIQQiffff", c.n_ops, c.compute_bytes, c.W, c.data_seed, w, opt["kind"], opt["lr"],
                       opt["beta1"], opt["beta2"], opt["eps"])
    out += np.asarray(c.meta["param_counts"], dtype=np.uint64).tobytes()
    for k in range(c.W):
        s = w + k
        out += struct.pack("<Q", s)
        for i in range(c.n_ops):
            o = c.op(s, i)
            out += struct.pack("<Q", o["step"])
            for name in ("master", "m", "v"):
                out += np.ascontiguousarray(o[name], dtype=np.float32).tobytes()
        a, co = c.slot(k)
        out += struct.pack("<I", len(a)) + np.asarray(a, dtype=np.uint32).tobytes()
        out += struct.pack("<I", len(co)) + np.asarray(co, dtype=np.uint32).tobytes()
    for it in range(w + 1, w + c.W + 1):
        for i in range(c.n_ops):
            out += np.ascontiguousarray(c.grads(it, i), dtype=np.float32).tobytes()
    with open(path, "wb") as fh:
        fh.write(out)


def test_shim_binary_exists():
    """Built by __graft_entry__.build() / `make -C tests/cpp` (CPU check)."""
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/shim_parity not built")
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("name,w", [("verify_toy", 3), ("six_op_cb1", 3), ("toy_sgd", 0)])
def test_cpp_shim_window_matches_reference(tmp_path, reference, name, w):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/shim_parity not built")
    c = load_case(name)
    case = tmp_path / "case.bin"
    write_case(c, w, case)
    res = subprocess.run([BIN, str(case), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr + res.stdout
    for k in range(c.W):
        assert (tmp_path / f"blob_{k}.bin").read_bytes() == c.blob(w + k), k
    assert (tmp_path / "conv.bin").read_bytes() == c.converted(w)
    out = res.stdout
    assert "ERR invalid_argument: snapshot slot references unknown operator" in out
    assert "ERR runtime_error: container checksum mismatch" in out
    assert f"ERR runtime_error: sparse checkpoint incomplete: 0 of {c.W + 1} records" in out
    assert f"PARSED iteration {w} entries" in out
    assert "complete 1 persisted 0" in out
    # window durability: the saved records load back byte-exact; a file copy is
    # one durable copy (persisted only at target 1); the ring promotes the window
    assert "SAVED same 1 durable_persisted 0" in out
    assert f"RING before 0 after {w} in_flight 0" in out
    # recovery from replica buffers: witnesses sent beside the replicas, records wrapped in place
    assert f"REPLICA_WITNESS same 1 witnessed {c.W} fallbacks 0" in out
    assert (tmp_path / "window" / f"window_{w}_slot_0.mlck").read_bytes() == c.blob(w)
    # conversion_plan, scalar codecs and the log budget through the C++ shim
    plan_line = next(x for x in out.splitlines() if x.startswith("PLAN "))
    want = [f"{k}:{it}:" + ",".join(str(i) for i in ids)
            for k, it, ids in ref_conversion_plan(reference, w, c.W, c.window_blobs(w), c.compute_bytes)]
    assert plan_line.split()[1:] == [str(w)] + want
    assert "CODEC inf 240 15360 1 " in out  # tensor.hpp: fp16 overflow, E4M3 saturation, 0x3c00
    assert "ERR invalid_argument: quantize: unsupported width 3" in out
    assert "LOGBYTES 38654705664" in out
    if name == "verify_toy":  # the GPU trainer as the gradient source: both conversions exact
        assert "ENGINE recompute 1 logged 1 log_entries " in out
        assert "SEGMENT ops 6 same 1" in out  # stage 1 of 3: one layer's 4 experts + NE + gate
        assert "ERR runtime_error: upstream log missing entry: iteration " in out
    assert "ERR invalid_argument: upstream log budget exceeded: need 38654705664 bytes of host memory, " \
           "budget 1000000000" in out
