"""Latency-model fit (cost_model.cpp:96-160): scls_fit_latency
is host code in the product library, so these run on CPU.  They restate the
reference's own fit tests (tests/cost_model_test.cpp:100-193 upstream) --
noiseless recovery to 1e-9, 1%-noise recovery to 5%, too few samples,
rank-deficient designs, models that go negative at the operating corner --
and compare with the reference's fit compiled here (oracle/_ref, which
solves through the normal equations of the Eigen stand-in; the predictions of
the two fits agree within the north star's 1e-9 relative tolerance)."""
import numpy as np
import pytest

from oracle.pyoracle import ref_lib
from paper_2406_13511_b200 import capi, lib
from paper_2406_13511_b200.lib import SclsError

SIZES = (1, 2, 4, 6, 8, 12, 16, 24, 32, 48, 64)
LENGTHS = (16, 32, 64, 128, 256, 384, 512, 768, 1024, 1536, 2048)


def reference_model():
    # cost_model_test.cpp reference_model(): the builtin profile of run_config.cpp
    return capi.builtin_latency_model()


def prefill(m, n, l):
    return m.p1 * n * l + m.p2 * n + m.p3 * l + m.p4


def decode_step(m, ctx, n):
    return m.d1 * n * ctx + m.d2 * n + m.d3 * ctx + m.d4


def synthesize(truth, noise_rel, seed):
    rng = np.random.default_rng(seed)
    out = []
    for n in SIZES:
        for l in LENGTHS:
            jp = 1.0 + noise_rel * (2.0 * rng.random() - 1.0)
            jd = 1.0 + noise_rel * (2.0 * rng.random() - 1.0)
            out.append(("prefill", n, l, prefill(truth, n, l) * jp))
            out.append(("decode", n, l, decode_step(truth, l, n) * jd))
    return out


def test_recovers_noiseless_model_to_float_precision():
    truth = reference_model()
    fitted = lib.fit_latency(synthesize(truth, 0.0, 1), truth.n_cap, truth.l_cap)
    assert fitted.rmse_prefill < 1e-9 and fitted.rmse_decode < 1e-9
    for n in (1, 5, 17, 64):
        for l in (1, 100, 999, 4096):
            assert abs(prefill(fitted, n, l) - prefill(truth, n, l)) < 1e-9
            assert abs(decode_step(fitted, l, n) - decode_step(truth, l, n)) < 1e-9


def test_recovers_coefficients_under_one_percent_noise():
    truth = reference_model()
    fitted = lib.fit_latency(synthesize(truth, 0.01, 20260815), truth.n_cap, truth.l_cap)
    for f in ("p1", "p2", "p3", "p4", "d1", "d2", "d3", "d4"):
        assert abs(getattr(fitted, f) - getattr(truth, f)) <= 0.05 * abs(getattr(truth, f)), f


def test_throws_when_a_phase_has_too_few_samples():
    truth = reference_model()
    few = [("prefill", 1, 100, prefill(truth, 1, 100)), ("prefill", 2, 100, prefill(truth, 2, 100)),
           ("prefill", 1, 200, prefill(truth, 1, 200))]
    with pytest.raises(SclsError) as e:
        lib.fit_latency(few)
    assert e.value.name == "InsufficientSamplesError"
    assert "prefill fit needs >= 4 samples spanning >= 2 batch sizes and >= 2 lengths, got 3 samples" in str(e.value)
    no_decode = [s for s in synthesize(truth, 0.0, 1) if s[0] == "prefill"]
    with pytest.raises(SclsError) as e:
        lib.fit_latency(no_decode)
    assert e.value.name == "InsufficientSamplesError" and "decode fit needs" in str(e.value)


def test_throws_on_rank_deficient_design():
    truth = reference_model()
    rows = []
    for v in (1, 2, 3, 4, 5):  # n == l on every row: the n and l columns are collinear
        rows.append(("prefill", v, v, prefill(truth, v, v)))
        rows.append(("decode", v, v, decode_step(truth, v, v)))
    with pytest.raises(SclsError) as e:
        lib.fit_latency(rows)
    assert e.value.name == "InsufficientSamplesError" and "rank-deficient" in str(e.value)


def test_rejects_models_predicting_negative_time():
    rows = []
    for n in (1, 2, 4, 8):
        for l in (16, 64, 256, 1024):
            v = 1.0 - 4e-4 * l
            rows.append(("prefill", n, l, v))
            rows.append(("decode", n, l, v))
    with pytest.raises(SclsError) as e:
        lib.fit_latency(rows, 64, 4096)
    assert e.value.name == "DegenerateModelError"


@pytest.mark.parametrize("noise", [0.0, 0.01, 0.2])
def test_matches_reference_fit(noise):
    ref = ref_lib()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    truth = reference_model()
    rows = synthesize(truth, noise, 7)
    a = lib.fit_latency(rows, truth.n_cap, truth.l_cap)
    b = ref.fit_latency(rows, truth.n_cap, truth.l_cap)
    for n in SIZES:
        for l in LENGTHS:
            for f in (prefill, lambda m, n_, l_: decode_step(m, l_, n_)):
                x, y = f(a, n, l), f(b, n, l)
                assert abs(x - y) <= 1e-9 * abs(y), (noise, n, l)
    assert abs(a.rmse_prefill - b.rmse_prefill) <= 1e-9 * max(b.rmse_prefill, 1e-12) + 1e-12
    assert abs(a.rmse_decode - b.rmse_decode) <= 1e-9 * max(b.rmse_decode, 1e-12) + 1e-12
    # the same errors on the same bad inputs
    with pytest.raises(Exception):
        ref.fit_latency(rows[:3])
