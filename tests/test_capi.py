"""The C-ABI boundary on CPU: the library loads, exports exactly what
include/scls_capi.h declares, its host-only helpers match the checker, and
without a GPU it refuses to compute (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2406_13511_b200 import capi, lib
from tests.conftest import ROOT
from tests.helpers import MEMORIES


def declared_functions():
    src = open(os.path.join(ROOT, "include", "scls_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scls_[a-z_0-9]+)\s*\(", src)))


def test_header_lists_match_binding():
    assert sorted(lib.EXPORTS) == declared_functions()


def test_library_exports_every_declared_symbol():
    L = lib.load()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = sorted(set(re.findall(r" T (scls_\w+)", out)))
    assert exported == declared_functions()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layouts():
    # sizes fixed by scls_capi.h (x86-64 SysV)
    assert C.sizeof(capi.Latency) == 8 * 10 + 8
    assert C.sizeof(capi.SchedCfg) == 6 * 4 + 3 * 8
    assert C.sizeof(capi.Memory) == 8 + 5 * 8 + 2 * 4 * capi.SCLS_MAX_RULES
    assert C.sizeof(capi.EventRecord) == 4 * 8 + 2 * 8 + 10 * 4 + 8
    assert C.sizeof(capi.Member) == 24


def test_validators_match_oracle(orc):
    L = lib.load()
    lats = [capi.builtin_latency_model(), capi.latency_model(p1=-1.0), capi.latency_model(),
            capi.latency_model(d4=float("nan")), capi.latency_model(p2=1.0, n_cap=0)]
    for m in lats:
        assert L.scls_validate_latency(C.byref(m)) == orc.validate_latency(m)
    mems = [MEMORIES["rule"](), MEMORIES["analytic"](), capi.analytic(1.0, 1.0, 1.0, 1.0),
            capi.analytic(10.0, 1.0, 1.0, 1.0, 1.5), capi.rule_table([(0, 5), (10, 3)]),
            capi.rule_table([(10, 5), (0, 3)]), capi.rule_table([(10, 0)])]
    for m in mems:
        assert L.scls_validate_memory(C.byref(m)) == orc.validate_memory(m)
    cfgs = [capi.sched_cfg(), capi.sched_cfg(lambda_=1.0), capi.sched_cfg(gamma=0.0),
            capi.sched_cfg(slice_len=0), capi.sched_cfg(slice_len=2048),
            capi.sched_cfg(fixed_batch_size=0), capi.sched_cfg(max_concurrent=0),
            capi.sched_cfg(worker_count=0)]
    for c in cfgs:
        assert L.scls_validate_sched(C.byref(c)) == orc.validate_sched(c)


def test_generate_matches_oracle(orc, golden):
    for g in golden["generate"]:
        spec = capi.workload_spec(rate=g["rate"], duration_s=g["duration_s"], seed=g["seed"])
        a = lib.generate(spec)
        b = orc.generate(spec)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for spec in (capi.workload_spec(input_dist=capi.uniform_dist(1, 1024), duration_s=50.0),
                 capi.workload_spec(gen_dist=capi.lognormal_dist(5.0, 1.0, 900), duration_s=50.0),
                 capi.workload_spec(gen_dist=capi.long_gen_dist(), duration_s=50.0, seed=9)):
        for x, y in zip(lib.generate(spec), orc.generate(spec)):
            assert np.array_equal(x, y)


def test_make_pool_matches_oracle(orc):
    for x, y in zip(lib.make_pool(4096, 7), orc.make_pool(4096, 7)):
        assert np.array_equal(x, y)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lib.SclsError) as e:
        lib.Context(0)
    assert e.value.status == capi.ERR_CUDA
