"""The measurement seam: B200 timings exported in the
reference's profile-CSV format must parse with the reference's own parser
and fit, and a PerfModel built from them must drive the reference-compatible
scheduler/driver.  GPU part: measure_perf_model times real prefills and decode
steps."""

import os
import sys

import pytest

from paper_2311_18677_b200.perf import PROFILE_HEADER, PerfModel, export_profile_csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _toy_b200_model():
    return PerfModel("B200", "llama2-7b", ([1, 512, 1024, 2048], [1.0, 8.0, 15.0, 31.0]),
                     ([1, 2, 4, 8, 16], [3.2, 3.6, 4.5, 5.0, 6.0]), 524288.0, 13.5e9, 180e9, 64)


def _reference():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "splitsim")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import splitsim
            return splitsim
    pytest.skip("reference package not available")


def test_profile_csv_roundtrips_through_reference_fit():
    ss = _reference()
    text = export_profile_csv(_toy_b200_model())
    assert text.splitlines()[0] == PROFILE_HEADER
    samples = ss.parse_profile_csv(text)
    assert len(samples) == 9
    model, report = ss.fit_piecewise_linear(samples, memory_capacity=180e9)
    assert model.prompt_time(1024) == pytest.approx(15.0)
    assert model.token_iter_time(4) == pytest.approx(4.5)
    assert report.train_mape_prompt < 1e-6


def test_b200_perf_model_drives_reference_simulator_and_ours():
    """Same B200 PerfModel in the reference Simulator and in our Driver:
    identical per-request TTFT/E2E for a Splitwise 1+1 layout."""
    ss = _reference()
    from paper_2311_18677_b200.cluster import ClusterConfig
    from paper_2311_18677_b200.driver import Driver, Request
    m = _toy_b200_model()
    ref_model = ss.PerfModel(m.machine_type, m.llm, m.prompt_knots, m.token_knots,
                             m.kv_bytes_per_token, m.weight_memory, m.memory_capacity,
                             m.max_token_batch)
    reqs = [(0, 0.0, 1024, 128), (1, 0.001, 1024, 128), (2, 0.02, 300, 20)]
    tr = ss.Trace([ss.Request(*r) for r in reqs], 1.0)
    tcfg = ss.TransferConfig(bandwidth=770e9 * 8, mode_threshold_tokens=33,
                             layerwise_constant_ms=0.05, num_layers=32)
    # the reference has no B200 machine type: register the B200 model under
    # the "H100" key of a Splitwise-HH layout (machine type only selects the model)
    res = ss.Simulator(ss.ClusterConfig("Splitwise-HH", 1, 1, transfer=tcfg),
                       {"H100": ref_model}, tr).run()
    from paper_2311_18677_b200.transfer import TransferConfig
    ours = Driver(ClusterConfig("Splitwise-HH", 1, 1,
                                transfer=TransferConfig(770e9 * 8, 33, 0.05, 32)),
                  {"H100": m}, [Request(*r) for r in reqs], duration_s=1.0).run()
    for rec in res.report.records:
        got = ours.records[rec.request.id]
        assert got.ttft_ms == pytest.approx(rec.ttft_ms)
        assert got.e2e_ms == pytest.approx(rec.e2e_ms)


@pytest.mark.gpu
def test_measure_perf_model_on_gpu():
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.model import get_config, init_weights
    from paper_2311_18677_b200.perf import measure_perf_model
    from paper_2311_18677_b200.runner import ModelRunner
    cfg = get_config("tiny")
    w = init_weights(cfg)
    kv = KVCacheManager(cfg.n_layers, 2048, cfg.n_kv_heads, cfg.head_dim, 16, 32, 256)
    m = measure_perf_model(ModelRunner(w, kv), prompt_points=(64, 256, 1024),
                           batch_points=(1, 2, 4), context=256, reps=2)
    assert m.prompt_time(256) > 0 and m.token_iter_time(2) > 0
    text = export_profile_csv(m)
    assert len(text.splitlines()) == 1 + 3 + 3
