"""Small invocations of every product kernel, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python scripts/sanitize.py [part ...]

Parts: fnv (TMA and byte paths, unaligned, multi-chunk look-back), pack
(snapshot of the verify_toy window under every transport, incl. the fused
gather kernel), convert (walk + replay), log (pinned-host and device rings),
codec.  Each result is checked against the committed goldens / the CPU
oracle, so a clean sanitizer log is also a parity pass.  Sizes are small:
the FNV grids stay below the SM count (look-back co-residency holds under
the tool's scheduling).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_cases import load_case  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2412_15411_b200 import mlck  # noqa: E402


def part_fnv(ctx, oracle):
    for n in (1, 127, 128, 129, 4096 + 3, 65536, 3 * 65536 + 5, 9 * 65536 + 77):
        data = np.random.default_rng(n).integers(0, 256, n + 16, dtype=np.uint8)
        p = ctx.upload(data)
        try:
            assert ctx.fnv1a64(p, n) == oracle.fnv1a64(data[:n]), n
            assert ctx.fnv1a64(p + 3, n) == oracle.fnv1a64(data[3:3 + n]), n
            assert ctx.fnv1a64(p + 16, n) == oracle.fnv1a64(data[16:16 + n]), n
        finally:
            ctx.free(p)
    print("fnv ok")


def _upload_state(ctx, c, s):
    st = mlck.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    for i in range(c.n_ops):
        o = c.op(s, i)
        st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
    st.set_meta(s, c.data_seed)
    return st


def part_pack(ctx, oracle):
    c = load_case("verify_toy")
    w = 3
    for mode in (0, 1, 2, 3, 4, 5):
        ctx.set_replica_mode(mode)
        for k in range(c.W):
            s = w + k
            st = _upload_state(ctx, c, s)
            b = mlck.Blob(ctx)
            rep = mlck.Blob(ctx, 1 << 16)
            b.add_replica(rep.device_ptr, 1 << 16)
            a, co = c.slot(k)
            mlck.snapshot_record(st, a, co, k, 1, w, c.W, out=b)
            got = b.to_host()
            assert got == c.blob(s), (mode, k)
            assert ctx.download(rep.device_ptr, len(got)) == got, (mode, k)
            b.close(), rep.close(), st.close()
    ctx.set_replica_mode(-1)
    # dense checkpoint + MLST image
    st = _upload_state(ctx, c, w)
    d = mlck.dense_checkpoint(st)
    assert int.from_bytes(d.to_host()[-8:], "little") == oracle.fnv1a64(d.to_host()[:-8])
    st.serialize_state()
    print("pack ok")


def part_convert(ctx, oracle):
    c = load_case("verify_toy")
    w = 3
    blobs = [mlck.Blob.from_host(ctx, c.blob(w + k)) for k in range(c.W)]
    g = mlck.GradLog(ctx, c.meta["param_counts"], c.W)
    for it in range(w + 1, w + c.W + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    out = mlck.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    mlck.sparse_to_dense_convert(out, blobs, w, c.W, c.data_seed, g)
    assert out.serialize_state() == c.converted(w)
    for b in blobs:
        mlck.parse_record(b, c.compute_bytes)
    mlck.check_coverage(blobs, c.n_ops, c.compute_bytes)
    print("convert ok")


def part_log(ctx, oracle):
    n = 4096 * 3 + 7
    src = np.random.default_rng(5).standard_normal(n).astype(np.float32)
    p = ctx.upload(src)
    for kind in (0, 1):
        log = mlck.UpstreamLog(ctx, 1 << 22, kind=kind, device=0)
        for it in range(3):
            for mb in range(2):
                log.put(it, mb, 0, 0, p, n)
                log.put(it, mb, 0, 1, p, n)
        log.sync()
        assert np.array_equal(log.at(2, 1, 0, 1), src)
        log.gc(2)
        assert len(log) == 4
        log.close()
    ctx.free(p)
    print("log ok")


def part_codec(ctx, oracle):
    x = np.random.default_rng(9).standard_normal(10007).astype(np.float32) * 100
    x[:4] = [np.inf, -np.inf, np.nan, 0.0]
    pin = ctx.upload(x)
    pq, pc, pd = ctx.alloc(x.nbytes), ctx.alloc(x.nbytes), ctx.alloc(x.nbytes)
    for cb in (1, 2, 4):
        ctx.quantize(pin, pq, x.size, cb)
        ctx.encode_compute(pin, pc, x.size, cb)
        ctx.decode_compute(pc, pd, x.size, cb)
        q = np.frombuffer(ctx.download(pq, x.nbytes), np.float32)
        d = np.frombuffer(ctx.download(pd, x.nbytes), np.float32)
        same = (q.view(np.uint32) == d.view(np.uint32)) | (np.isnan(q) & np.isnan(d))
        assert same.all(), cb  # decode(encode(x)) == quantize(x)
    ctx.synchronize()
    for p in (pin, pq, pc, pd):
        ctx.free(p)
    print("codec ok")


PARTS = {"fnv": part_fnv, "pack": part_pack, "convert": part_convert, "log": part_log, "codec": part_codec}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    ctx = mlck.Context(0)
    oracle = Oracle()
    for nm in names:
        PARTS[nm](ctx, oracle)
    ctx.synchronize()
    print("sanitize driver done")
