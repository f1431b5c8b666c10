"""Device trace generation: generate() on the B200,
bit-exact with the reference's sampler (workload.cpp:100-181).

CPU tests pin the ingredients the device cannot take from the reference: the
ports of glibc 2.39's FMA-variant `log` (csrc/glibc_log.cuh, constants from
tools/extract_glibc_log.py) and `exp` / `cos` (csrc/glibc_expcos.cuh,
tools/extract_glibc_expcos.py), compiled for the host and compared bit for
bit with this image's libm over tens of millions of inputs, and the
log-normal draw against the reference's expression.  GPU tests compare the device port
with libm, scls_generate_batch with the host generator and the compiled
reference, and scls_run_sweep with scls_simulate_grid on host-generated
traces (every TraceResult field)."""
import ctypes as C
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2406_13511_b200 import capi
from tests.conftest import ROOT
from tests.helpers import MEMORIES

CSRC = os.path.join(ROOT, "paper_2406_13511_b200", "csrc")

CHECK_SRC = r"""
#include "glibc_log.cuh"
#include <cmath>
#include <cstdio>
#include <random>
int main() {
  std::mt19937_64 g(1);
  long bad = 0, n = 0;
  auto chk = [&](double x) {
    const double a = std::log(x), b = scls_glibc::log_fma(x);
    ++n;
    if (scls_glibc::f_bits(a) != scls_glibc::f_bits(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 5) std::printf("x=%a libm=%a port=%a\n", x, a, b);
      ++bad;
    }
  };
  for (int i = 0; i < 20000000; ++i) chk(1.0 - (double)(g() >> 11) * 0x1p-53);   // the sampler's domain
  for (int i = 0; i < 5000000; ++i) chk(0.93 + (double)(g() >> 11) * 0x1p-53 * 0.15);  // near-1 path
  for (int i = 0; i < 5000000; ++i) chk(scls_glibc::f_dbl(g()));                 // every bit pattern
  for (double x : {0.0, -0.0, 1.0, (double)INFINITY, -1.0, (double)NAN, 0x1p-1074, 0x1p-1060, 0x1p-53, 0x1.fffffffffffffp-1})
    chk(x);
  std::printf("n=%ld bad=%ld\n", n, bad);
  return bad != 0;
}
"""

LIBM_SRC = r"""
#include <math.h>
#include <stdint.h>
void libm_log(int64_t n, const double* x, double* y) { for (int64_t i = 0; i < n; ++i) y[i] = log(x[i]); }
"""


def _build(src, name, shared=False):
    d = tempfile.mkdtemp(prefix="scls_glog_")
    path = os.path.join(d, name + (".cpp" if not shared else ".c"))
    with open(path, "w") as f:
        f.write(src)
    out = os.path.join(d, name + (".so" if shared else ""))
    cmd = (["gcc", "-O2", "-shared", "-fPIC", path, "-o", out, "-lm"] if shared else
           ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", CSRC, path, "-o", out])
    subprocess.run(cmd, check=True, capture_output=True)
    return out


EXPCOS_SRC = r"""
#include "glibc_expcos.cuh"
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>
// the reference's log-normal draw (workload.cpp:112-118,136-141), on libm
static int ref_lognormal(double mu, double sigma, int cap, int limit, std::mt19937_64& e) {
  const double u1 = 1.0 - (double)(e() >> 11) * 0x1.0p-53;
  const double u2 = (double)(e() >> 11) * 0x1.0p-53;
  const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
  const double raw = std::exp(mu + sigma * z);
  const long long rounded = raw > 1e18 ? (long long)1e18 : std::llround(raw);
  const long long v = std::min<long long>(rounded, cap);
  return v < 1 ? 1 : (v > limit ? limit : (int)v);
}
int main() {
  using namespace scls_glibc;
  std::mt19937_64 g(1);
  long bad = 0, n = 0;
  auto chk = [&](const char* f, double x, double a, double b) {
    ++n;
    if (f_bits(a) != f_bits(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 5) std::printf("%s(%a) libm=%a port=%a\n", f, x, a, b);
      ++bad;
    }
  };
  auto u = [&]() { return (double)(g() >> 11) * 0x1p-53; };
  for (int i = 0; i < 8000000; ++i) { const double x = 6.283185307179586 * u(); chk("cos", x, std::cos(x), cos_fma(x)); }
  for (int i = 0; i < 2000000; ++i) { const double x = 0.9 * u(); chk("cos", x, std::cos(x), cos_fma(x)); }
  for (int i = 0; i < 2000000; ++i) { const double x = 1e-6 * u(); chk("cos", x, std::cos(x), cos_fma(x)); }
  for (int i = 0; i < 2000000; ++i) { const double x = (u() - 0.5) * 2e6; chk("cos", x, std::cos(x), cos_fma(x)); }
  for (int i = 0; i < 8000000; ++i) { const double x = (u() - 0.5) * 100.0; chk("exp", x, std::exp(x), exp_fma(x)); }
  for (int i = 0; i < 2000000; ++i) { const double x = (u() - 0.5) * 1023.0; chk("exp", x, std::exp(x), exp_fma(x)); }
  for (int i = 0; i < 2000000; ++i) { const double x = (u() - 0.5) * 1e-3; chk("exp", x, std::exp(x), exp_fma(x)); }
  for (double x : {0.0, -0.0, 1e-300, 0x1p-27, 0x1p-28, 0.855469, 2.426265, 3.14159, 6.283185307179586})
    chk("cos", x, std::cos(x), cos_fma(x));
  for (double x : {0.0, -0.0, 1e-300, 0x1p-54, 0x1p-55, 1.0, 41.44653167389282, 41.4465316738928, 511.9, -511.9})
    chk("exp", x, std::exp(x), exp_fma(x));
  // the sampler end to end: mu / sigma spread incl. raw beyond 1e18 and below 0.5
  const double mus[] = {-2.0, 0.0, 3.0, 5.5, 6.2, 7.0, 40.0, 45.0};
  const double sig[] = {0.1, 0.5, 1.0, 2.0, 10.0};
  for (double mu : mus)
    for (double s : sig) {
      std::mt19937_64 a(123), b(123);
      for (int i = 0; i < 100000; ++i) {
        const int r = ref_lognormal(mu, s, 1 << 30, 1 << 30, a);
        const uint64_t w0 = b(), w1 = b();
        ++n;
        if (r != lognormal_length(mu, s, 1 << 30, 1 << 30, w0, w1)) ++bad;
      }
    }
  std::printf("n=%ld bad=%ld\n", n, bad);
  return bad != 0;
}
"""


def test_glibc_expcos_port_matches_libm_on_host():
    """csrc/glibc_expcos.cuh (host build) == this image's libm exp / cos, bit
    for bit, and the log-normal draw == the reference's expression on libm."""
    d = tempfile.mkdtemp(prefix="scls_gexp_")
    src, exe = os.path.join(d, "c.cpp"), os.path.join(d, "c")
    with open(src, "w") as f:
        f.write(EXPCOS_SRC)
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-I", CSRC, src, "-o", exe],
                   check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    assert "bad=0" in r.stdout


def test_expcos_tables_match_this_libm(tmp_path):
    import importlib.util
    spec = importlib.util.spec_from_file_location("extract2", os.path.join(ROOT, "tools", "extract_glibc_expcos.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.OUT = str(tmp_path / "glibc_expcos_data.h")
    mod.main()
    want = open(os.path.join(CSRC, "glibc_expcos_data.h")).read().split("\n", 1)[1]
    got = open(mod.OUT).read().split("\n", 1)[1]
    assert got == want


def test_glibc_log_port_matches_libm_on_host():
    exe = _build(CHECK_SRC, "glog_check")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    assert "bad=0" in r.stdout


def test_log_table_matches_this_libm(tmp_path):
    """The committed constants are the ones this image's libm carries."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("extract", os.path.join(ROOT, "tools", "extract_glibc_log.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.OUT = str(tmp_path / "glibc_log_data.h")
    mod.main()
    want = open(os.path.join(CSRC, "glibc_log_data.h")).read().split("\n", 1)[1]
    got = open(mod.OUT).read().split("\n", 1)[1]
    assert got == want


# ------------------------------------------------------------------------------------------
def _specs():
    """A spread of WorkloadSpecs: histogram (codefuse-like, long-gen) and
    uniform lengths, tight limits, tiny and empty traces, many seeds/rates."""
    out = []
    for i in range(48):
        out.append(capi.workload_spec(rate=float(1 + i % 25), duration_s=float(20 + 13 * (i % 7)), seed=7000 + i))
    out.append(capi.workload_spec(rate=20.0, duration_s=600.0, seed=42))
    out.append(capi.workload_spec(rate=2.0, duration_s=500.0, seed=42))
    out.append(capi.workload_spec(rate=5.0, duration_s=0.0, seed=1))           # empty trace
    out.append(capi.workload_spec(rate=0.01, duration_s=3.0, seed=3))          # almost surely empty
    out.append(capi.workload_spec(rate=50.0, duration_s=100.0, gen_dist=capi.long_gen_dist(), seed=9))
    u = capi.uniform_dist(1, 2000)
    out.append(capi.workload_spec(rate=30.0, duration_s=100.0, input_dist=u, gen_dist=capi.uniform_dist(5, 700),
                                  max_input_limit=1500, max_gen_limit=300, seed=11))
    out.append(capi.workload_spec(rate=8.0, duration_s=200.0, input_dist=u, seed=2 ** 63 + 5))
    out.append(capi.workload_spec(rate=1000.0, duration_s=30.0, max_input_limit=100, max_gen_limit=50, seed=0))
    # log-normal lengths (Box-Muller: two outputs per draw), mixed with the other kinds
    ln = capi.lognormal_dist(5.0, 1.0, 900)
    out.append(capi.workload_spec(rate=10.0, duration_s=100.0, gen_dist=ln, seed=21))
    out.append(capi.workload_spec(rate=15.0, duration_s=80.0, input_dist=capi.lognormal_dist(6.0, 0.8, 2000),
                                  gen_dist=capi.lognormal_dist(4.5, 1.5, 4096), max_gen_limit=700, seed=22))
    out.append(capi.workload_spec(rate=12.0, duration_s=60.0, input_dist=capi.lognormal_dist(3.0, 2.5, 1 << 30),
                                  gen_dist=u, seed=23))
    return out


@pytest.mark.gpu
def test_device_log_matches_libm(ctx):
    so = _build(LIBM_SRC, "libm_log", shared=True)
    libm = C.CDLL(so)
    libm.libm_log.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(5)
    u = (rng.integers(0, 2 ** 53, 4_000_000, dtype=np.int64).astype(np.float64)) * 2.0 ** -53
    x = np.concatenate([1.0 - u, 0.93 + 0.15 * u[:1_000_000],
                        rng.integers(0, 2 ** 63, 1_000_000, dtype=np.int64).view(np.float64),
                        np.array([0.0, -0.0, 1.0, np.inf, -1.0, np.nan, 5e-324, 2.0 ** -1060, 2.0 ** -53])])
    want = np.zeros_like(x)
    libm.libm_log(len(x), x.ctypes.data, want.ctypes.data)
    got = ctx.debug_log(x)
    nan = np.isnan(want) & np.isnan(got)
    bad = (got.view(np.int64) != want.view(np.int64)) & ~nan
    assert not bad.any(), (x[bad][:5], got[bad][:5], want[bad][:5])


@pytest.mark.gpu
def test_device_exp_cos_match_libm(ctx):
    """The device ports of glibc exp / cos (the log-normal draw) == libm."""
    so = _build(LIBM_SRC + r"""
void libm_exp(int64_t n, const double* x, double* y) { for (int64_t i = 0; i < n; ++i) y[i] = exp(x[i]); }
void libm_cos(int64_t n, const double* x, double* y) { for (int64_t i = 0; i < n; ++i) y[i] = cos(x[i]); }
""", "libm_ec", shared=True)
    libm = C.CDLL(so)
    rng = np.random.default_rng(11)
    u = (rng.integers(0, 2 ** 53, 3_000_000, dtype=np.int64).astype(np.float64)) * 2.0 ** -53
    cases = {"cos": np.concatenate([2 * np.pi * u, 0.9 * u[:500_000], 1e-6 * u[:200_000],
                                    (u[:500_000] - 0.5) * 2e6, [0.0, -0.0, 2.0 ** -27, 2.0 ** -28, 0.855469, 2.426265]]),
             "exp": np.concatenate([(u - 0.5) * 100.0, (u[:500_000] - 0.5) * 1023.0, (u[:200_000] - 0.5) * 1e-3,
                                    [0.0, -0.0, 2.0 ** -54, 2.0 ** -55, 1.0, 41.44653167389282, 511.9, -511.9]])}
    for fn, x in cases.items():
        f = getattr(libm, "libm_" + fn)
        f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
        want = np.zeros_like(x)
        f(len(x), x.ctypes.data, want.ctypes.data)
        got = ctx.debug_libm(fn, x)
        bad = got.view(np.int64) != want.view(np.int64)
        assert not bad.any(), (fn, x[bad][:5], got[bad][:5], want[bad][:5])


@pytest.mark.gpu
def test_device_lognormal_generation_large(ctx, orc):
    """2M log-normal draws on the device (1M requests, both lengths log-normal)
    == the compiled reference's generate(), request by request."""
    from oracle import pyoracle
    from paper_2406_13511_b200 import lib
    ref = pyoracle.ref_lib()
    specs = [capi.workload_spec(rate=1000.0, duration_s=1000.0, input_dist=capi.lognormal_dist(6.0, 1.2, 8192),
                                gen_dist=capi.lognormal_dist(5.0, 1.0, 4096), max_input_limit=4096,
                                max_gen_limit=2048, seed=77),
             capi.workload_spec(rate=200.0, duration_s=500.0, input_dist=capi.lognormal_dist(44.0, 3.0, 1 << 30),
                                gen_dist=capi.lognormal_dist(-1.0, 4.0, 1 << 30), seed=78)]
    offs, arr, inp, gen = ctx.generate_batch(specs)
    for t, sp in enumerate(specs):
        want = (ref or orc).generate(sp)
        lo, hi = offs[t], offs[t + 1]
        assert hi - lo == len(want[0]), t
        assert np.array_equal(arr[lo:hi].view(np.int64), np.asarray(want[0], np.float64).view(np.int64)), t
        assert np.array_equal(inp[lo:hi], want[1]) and np.array_equal(gen[lo:hi], want[2]), t


@pytest.mark.gpu
def test_generate_batch_matches_host_and_reference(ctx, orc):
    from oracle import pyoracle
    from paper_2406_13511_b200 import lib
    ref = pyoracle.ref_lib()
    specs = _specs()
    offs, arr, inp, gen = ctx.generate_batch(specs)
    for t, sp in enumerate(specs):
        a, b, g = lib.generate(sp)  # host generator (std::log)
        lo, hi = offs[t], offs[t + 1]
        assert hi - lo == len(a), t
        assert np.array_equal(arr[lo:hi].view(np.int64), np.asarray(a).view(np.int64)), t
        assert np.array_equal(inp[lo:hi], b) and np.array_equal(gen[lo:hi], g), t
        want = (ref or orc).generate(sp)
        assert np.array_equal(arr[lo:hi].view(np.int64), np.asarray(want[0], np.float64).view(np.int64)), t
        assert np.array_equal(inp[lo:hi], want[1]) and np.array_equal(gen[lo:hi], want[2]), t


@pytest.mark.gpu
def test_generate_batch_large_sweep_fingerprint(ctx):
    """The bench's C5 traces (1024 seeds x 4 rates, 600 s): device == host, all 4096."""
    from paper_2406_13511_b200 import lib
    specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4)
             for i in range(4096)]
    offs, arr, inp, gen = ctx.generate_batch(specs)
    rng = np.random.default_rng(0)
    for t in sorted(set(rng.integers(0, 4096, 64).tolist()) | {0, 4095}):
        a, b, g = lib.generate(specs[t])
        lo, hi = offs[t], offs[t + 1]
        assert hi - lo == len(a)
        assert np.array_equal(arr[lo:hi].view(np.int64), np.asarray(a).view(np.int64))
        assert np.array_equal(inp[lo:hi], b) and np.array_equal(gen[lo:hi], g)
    assert ctx.timings()["generate"] > 0


@pytest.mark.gpu
def test_run_sweep_equals_simulate_grid(ctx):
    from paper_2406_13511_b200 import lib
    lat, mem = capi.builtin_latency_model(), MEMORIES["rule"]()
    specs = _specs()
    cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")] + \
           [capi.sched_cfg(policy="scls", slice_len=64, worker_count=3, max_gen_limit=512)]
    a, ha = ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
    traces = [lib.generate(s) for s in specs]
    b, hb = ctx.simulate_grid(traces, cfgs, lat, mem, hist_bins=16)
    n = len(specs)
    for c in range(len(cfgs)):
        for t in range(n):
            for f, _ in capi.TraceResult._fields_:
                assert getattr(a[c * n + t], f) == getattr(b[c][t], f), (c, t, f)
    assert np.array_equal(ha, hb)


@pytest.mark.gpu
def test_run_sweep_errors(ctx):
    lat, mem = capi.builtin_latency_model(), MEMORIES["rule"]()
    from paper_2406_13511_b200.lib import SclsError
    bad = capi.workload_spec(rate=-1.0)
    with pytest.raises(SclsError) as e:
        ctx.run_sweep([bad], [capi.sched_cfg(policy="scls")], lat, mem)
    assert e.value.name == "Error" and "rate" in str(e.value)
    bad = capi.workload_spec(rate=5.0, duration_s=10.0, gen_dist=capi.lognormal_dist(5.0, -1.0, 1024))
    with pytest.raises(SclsError) as e:
        ctx.run_sweep([bad], [capi.sched_cfg(policy="scls")], lat, mem)
    assert e.value.name == "Error"


@pytest.mark.gpu
def test_run_experiments_equals_simulate(ctx):
    """experiment.cpp sweep body: run i = generate(specs[i]) under cfgs[i]."""
    from paper_2406_13511_b200 import lib
    lat, mem = capi.builtin_latency_model(), MEMORIES["rule"]()
    specs = _specs()
    pols = ("scls", "sls", "ils")
    cfgs = [capi.sched_cfg(policy=pols[i % 3], slice_len=(32, 64, 128, 256)[i % 4],
                           worker_count=1 + i % 8, max_gen_limit=512 if i % 4 < 3 else 1024)
            for i in range(len(specs))]
    a, ha = ctx.run_experiments(specs, cfgs, lat, mem, hist_bins=40)
    traces = [lib.generate(s) for s in specs]
    b, hb = ctx.simulate(traces, cfgs, lat, mem, cfg_index=list(range(len(specs))), hist_bins=40)
    for t in range(len(specs)):
        for f, _ in capi.TraceResult._fields_:
            assert getattr(a[t], f) == getattr(b[t], f), (t, f)
    assert np.array_equal(ha, hb)


@pytest.mark.gpu
def test_run_sweep_statuses_match_reference(ctx, orc):
    """Device-generated sweeps carry the reference's failure statuses:
    NonTermination (short horizon), InfeasibleRequest (a KV cap no request
    fits), EmptyLog (no arrivals), per job, next to healthy jobs."""
    from oracle import pyoracle
    ref = pyoracle.ref_lib() or orc
    lat = capi.builtin_latency_model()
    specs = [capi.workload_spec(rate=15.0, duration_s=120.0, seed=5),
             capi.workload_spec(rate=5.0, duration_s=0.0, seed=6),
             capi.workload_spec(rate=30.0, duration_s=200.0, seed=7)]
    for mem, cfgs in ((MEMORIES["rule"](), [capi.sched_cfg(policy=p, horizon_s=h) for p in ("scls", "sls", "ils")
                                            for h in (1e7, 30.0)]),
                      (capi.analytic(1000.0, 3.0, 2.0, 1.0, 1.0), [capi.sched_cfg(policy="scls")])):
        ctx.set_digests(False)
        try:
            a, _ = ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
        finally:
            ctx.set_digests(True)
        traces = [ref.generate(s) for s in specs]
        n = len(specs)
        statuses = set()
        for c, cfg in enumerate(cfgs):
            b, _ = ref.simulate(traces, cfg, lat, mem, hist_bins=16)
            for t in range(n):
                statuses.add(b[t].status)
                for f, _ in capi.TraceResult._fields_:
                    if not f.startswith("h_") and f != "sim_clock":
                        assert getattr(a[c * n + t], f) == getattr(b[t], f), (c, t, f)
        assert len(statuses) >= 2, statuses
