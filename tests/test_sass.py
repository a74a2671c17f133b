"""Static SASS checks of the built library (no GPU): the instructions the
design relies on are really in the kernels, and nothing ptxas inserted undoes
the look-back's latency work.

- fnv_kernel (every instantiation): TMA tensor loads and stores (UTMALDG /
  UTMASTG), mbarrier waits (SYNCS.PHASECHK) and the u8 IMMA final pass
  (DESIGN 3.1, 3.2).
- fnv_witness_tc_kernel: tcgen05 integer MMAs (UTCIMMA) with tcgen05.commit
  (UTCBAR) and a TMA load (DESIGN 3.3).
- fnv_kernel's YIELDs sit only in the out-of-line mbarrier retry stubs (each
  directly before a SYNCS.PHASECHK): a YIELD at a look-back loop head cost ~8 %
  of the kernel (DESIGN 3.2, staggered-start A/B).
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2412_15411_b200", "_build", "kernels.o")

pytestmark = pytest.mark.skipif(not (os.path.exists(OBJ) and shutil.which("cuobjdump")),
                                reason="library not built or cuobjdump missing")


@pytest.fixture(scope="module")
def kernels():
    text = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
    out, name = {}, None
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            out[name] = []
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and name:
            out[name].append(m.group(1))
    return out


def _find(kernels, key):
    found = {k: v for k, v in kernels.items() if key in k}
    assert found, f"no {key} in {OBJ}"
    return found


def _count(ops, prefix):
    return sum(1 for o in ops if o == prefix or o.startswith(prefix + "."))


def test_fnv_kernel_uses_tma_mbarriers_and_imma(kernels):
    for name, ops in _find(kernels, "fnv_kernel").items():
        assert _count(ops, "UTMASTG") > 0, name
        assert _count(ops, "SYNCS.PHASECHK") > 0, name
        assert _count(ops, "IMMA") > 0, name
    fused = [ops for k, ops in _find(kernels, "fnv_kernel").items() if "ILb0ELb1E" in k]
    assert fused and _count(fused[0], "UTMALDG") > 0


def test_witness_verifier_runs_on_tcgen05(kernels):
    ops = next(iter(_find(kernels, "fnv_witness_tc_kernel").values()))
    assert _count(ops, "UTCIMMA") > 0
    assert _count(ops, "UTCBAR") > 0
    assert _count(ops, "UTMALDG") > 0


def test_fnv_kernel_yields_only_in_retry_stubs(kernels):
    for name, ops in _find(kernels, "fnv_kernel").items():
        for i, o in enumerate(ops):
            if o == "YIELD":
                assert i + 1 < len(ops) and ops[i + 1].startswith("SYNCS.PHASECHK"), \
                    f"{name}: YIELD at instruction {i} is not an mbarrier retry stub"
