"""The device trace generator (ss_generate_traces_device) reproduces the host
generator (itself checked against the reference's generate() +
predictor_pipeline() in test_host.py) field for field, and the schedules it
feeds are the same."""

import numpy as np
import pytest

from paper_2506_12204_b200.predictors import PredictorConfig, Strategy
from paper_2506_12204_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu

CASES = [
    (WorkloadSpec(total_requests=1000), PredictorConfig()),
    (WorkloadSpec(total_requests=700, levels=3, urgency_weights=[1, 2, 3], gap_s=0.05), PredictorConfig()),
    (WorkloadSpec(total_requests=500, concurrent=500, concurrent_mode="fixed"), PredictorConfig()),
    (WorkloadSpec(total_requests=800, levels=4, output_len_range=(1, 300)),
     PredictorConfig(latency_s=0.01, batch_size=4, urgency_error=0.3, length_error=0.3)),
    (WorkloadSpec(total_requests=600), PredictorConfig(latency_s=0.02, batch_size=8,
                                                       strategy=Strategy.FULL_BATCHING, urgency_error=0.5)),
]


@pytest.mark.parametrize("k", range(len(CASES)))
def test_device_generator_matches_host(k):
    import torch

    from paper_2506_12204_b200.tracegen import generate_batch, generate_batch_device

    spec, pred = CASES[k]
    seeds = np.arange(100 * k, 100 * k + 64)
    host = generate_batch(spec, seeds, pred, pred_seeds=seeds + 7)
    dev = generate_batch_device(spec, seeds, pred, pred_seeds=seeds + 7)
    torch.cuda.synchronize()
    for f in ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie", "ids",
              "record_pos"):
        a = getattr(host, f)
        b = dev.t[f].cpu().numpy()[: len(a)].view(a.dtype) if a.dtype != np.float64 else dev.t[f].cpu().numpy()
        assert np.array_equal(a.view(np.uint8), np.ascontiguousarray(b[: len(a)]).view(np.uint8)), f


def test_device_generated_inputs_schedule_identically():
    import torch

    from paper_2506_12204_b200 import _abi as A
    from paper_2506_12204_b200 import native
    from paper_2506_12204_b200.costs import get_profile
    from paper_2506_12204_b200.results import make_params
    from paper_2506_12204_b200.tracegen import generate_batch, generate_batch_device

    spec = WorkloadSpec(total_requests=1000)
    seeds = np.arange(256)
    p = lambda: make_params(get_profile("a100_qwen7b"), 16, 10**9, flags=A.SS_FLAG_DIGEST)
    dev = torch.device("cuda", 0)
    runs = []
    for db in (native.DeviceBatch(generate_batch(spec, seeds), dev), generate_batch_device(spec, seeds)):
        outs = native.DeviceOutputs(db.n_requests, db.n_traces, dev, with_state=False)
        ws = native.Workspace(p(), db.n_traces, db.n_requests, dev)
        native.run_device(p(), db, outs, ws)
        runs.append(outs.stats_numpy())
    assert np.array_equal(runs[0]["digest"], runs[1]["digest"])
    assert np.array_equal(runs[0]["rounds"], runs[1]["rounds"])
