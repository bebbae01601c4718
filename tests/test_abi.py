"""The C-ABI library: builds for sm_100a, loads, exports every symbol that
include/gatewave_b200.h declares, and fails loudly (no CPU fallback) when no
GPU is present.  No compute calls here."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "gatewave_b200.h")).read()
    return sorted(set(re.findall(r"\b(gw_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2306_11006_b200 import build, engine
    build.build()
    lib = engine.load_library()
    decl = _declared()
    assert len(decl) >= 25
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(engine.EXPORTS) == decl


def test_library_is_sm100a():
    import subprocess
    from paper_2306_11006_b200 import engine
    out = subprocess.run(["cuobjdump", "--list-elf", engine.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_fft_kernel_has_no_local_memory_arrays():
    """ptxas report of the N=1024 blind rotation: no large stack frame."""
    info = open(os.path.join(ROOT, "paper_2306_11006_b200", "ptxas_info.txt")).read()
    m = re.search(r"k_blind_rotateILi10ELi2E.*?\n\s+(\d+) bytes stack frame", info, re.S)
    assert m and int(m.group(1)) <= 64


def test_no_gpu_means_loud_failure():
    from paper_2306_11006_b200 import engine
    if engine.device_count() > 0:
        pytest.skip("a GPU is visible")
    from conftest import MINI
    from paper_2306_11006_b200.cggi import GateKind, eval_gate_batch, keygen
    ks = keygen(MINI, 1)
    rows = np.zeros((1, MINI.n + 1), np.uint32)
    with pytest.raises(engine.EngineUnavailable):
        eval_gate_batch(GateKind.NAND, [rows, rows], ks.eval_key())
