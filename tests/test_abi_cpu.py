"""CPU checks of the product library: it loads, exports exactly the C ABI that
include/fbgpu.h declares, its host-side trace generation matches the
reference, and device entry points fail loudly (never fall back to the CPU)
when no GPU is present."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from catalog import TRACE_PROFILES, rows_digest
from paper_2510_14392_b200 import _abi, fbgpu
from paper_2510_14392_b200.batch import Batch, ms_to_us
from paper_2510_14392_b200 import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fbgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    fbgpu.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", fbgpu.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fb_[a-z_0-9]+)$", out, flags=re.M))
    declared = declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_abi_version_and_struct_sizes():
    L = fbgpu.lib()
    assert L.fb_abi_version() == 1
    import ctypes as C
    assert C.sizeof(_abi.Instance) == 8 * 3 + 4 * 2 + 8 + 8 * 3 + 8 + 8 + 8 * 2 + 4 * 2 + 8 * 3
    assert _abi.RECORD_DTYPE.itemsize == 32


@pytest.mark.parametrize("name", sorted(TRACE_PROFILES))
def test_host_trace_generation_matches_reference(golden, name):
    prof, h = TRACE_PROFILES[name]
    rows = fbgpu.generate_bursty(prof, ms_to_us(h))
    g = golden["traces"][name]
    assert len(rows) == g["n"] and rows_digest(rows) == g["sha256"]


def test_scale_trace_matches_python(oracle):
    rows = workloads.c1_rows()
    for f in (0.5, 1.5, 3.0, 7.0 / 3.0):
        a = fbgpu.scale_trace(rows, f).arrival_us
        assert np.array_equal(a, rows.scaled(f).arrival_us)
        assert np.array_equal(a, oracle.scale_trace(rows.arrival_us, f))


def test_generate_bursty_validation():
    bad = fbgpu.burst_profile(5.0, 1.0, 100, 100, 10, 20, 10, 20, 1)  # burst < base
    with pytest.raises(fbgpu.ValidationError):
        fbgpu.generate_bursty(bad, 1000)


def test_no_gpu_fails_loudly():
    if fbgpu.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(fbgpu.CudaError):
        fbgpu.Arena(0)
    with pytest.raises(fbgpu.CudaError):
        fbgpu.run_batch(workloads.c1_batch())


def test_workload_shapes():
    assert len(workloads.c1_rows()) == 931
    b = workloads.c2_batch(n_seeds=4)
    assert b.n_instances == 8 and b.instance(0).trace_off == b.instance(1).trace_off
    b3 = workloads.c3_batch(n_seeds=1, scales=workloads.C3_SCALES[:2], ttfts=(500.0,),
                            tpots=(50.0, 100.0))
    assert b3.n_instances == 2 * 2 * 4
    full = 64 * len(workloads.C3_SCALES) * 4 * 4 * 4
    assert full == 65_536
    s0 = workloads.c3_batch(n_seeds=1, scales=workloads.C3_SCALES[:2], ttfts=(500.0,),
                            tpots=(50.0,), shard=0, n_shards=2)
    s1 = workloads.c3_batch(n_seeds=1, scales=workloads.C3_SCALES[:2], ttfts=(500.0,),
                            tpots=(50.0,), shard=1, n_shards=2)
    assert s0.n_instances + s1.n_instances == 8
