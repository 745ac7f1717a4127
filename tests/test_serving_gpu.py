"""Batched unified draft/verify driver on the B200 (fp32 parity mode).

The token-level serving loop batches all draft and verify members of an
iteration into one forward; its per-request outputs must equal the
reference's plain greedy decode (golden streams from the reference,
configs[0]: 4 requests x 256-token prompt x 1024 tokens, k=4, s=0.05).
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2512_01278_b200 import model as M  # noqa: E402
from paper_2512_01278_b200.scheduler import PipelineMode  # noqa: E402
from paper_2512_01278_b200.simulate import KvPoolConfig, SimConfig, run_token_sim  # noqa: E402
from paper_2512_01278_b200.workload import LengthDist, LengthSpec, WorkloadSpec  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
C0_PLANTED = list(range(5, 256, 21))[:12]


def _workload(n, inp, out, seed=0):
    return WorkloadSpec(n_requests=n, input_len=LengthSpec(LengthDist.CONSTANT, inp),
                        output_len=LengthSpec(LengthDist.CONSTANT, out), seed=seed)


@pytest.mark.parametrize("tag,pipeline", [("c0", PipelineMode.DELAYED), ("c0p", PipelineMode.SYNCHRONOUS)])
def test_token_sim_configs0_matches_reference_streams(golden_streams, tag, pipeline):
    cfg = M.ModelConfig(2, 8, 2, 32, 512, seed=0)
    model = M.init_model(cfg)
    if tag == "c0p":
        model = M.plant_attention_concentration(model, C0_PLANTED)
    rep = run_token_sim(_workload(4, 256, 1024), cfg, SimConfig(k=4, alpha=0.0, sparsity=0.05, max_batch=4,
                                                               pipeline=pipeline),
                        KvPoolConfig(capacity_pages=1 << 16, page_bytes=64), model=model)
    gold = {c["rid"]: c["tokens"] for c in golden_streams if c.get("tag") == tag}
    assert set(rep.outputs) == set(gold)
    for rid, toks in gold.items():
        assert rep.outputs[rid] == toks, f"{tag} request {rid} diverged"
    assert rep.emitted_tokens == 4 * 1024
    if tag == "c0p":
        assert rep.realized_alpha == 1.0


def test_token_sim_lossless_small_mixed_lengths():
    cfg = M.ModelConfig(2, 4, 2, 8, 48, seed=3)
    wl = WorkloadSpec(n_requests=9, input_len=LengthSpec(LengthDist.NORMAL, 14, 5),
                      output_len=LengthSpec(LengthDist.NORMAL, 40, 15), seed=5)
    rep = run_token_sim(wl, cfg, SimConfig(k=3, alpha=0.0, sparsity=0.3, max_batch=4),
                        KvPoolConfig(capacity_pages=4096, page_bytes=64), check_lossless=True)
    assert len(rep.requests) == 9
    assert all(r.emitted >= 1 for r in rep.requests)
    # delayed mode: every verification but the last is followed by exactly one stall
    for r in rep.requests:
        assert r.stall_absences == max(0, r.rounds - 1)
    assert sum(rep.acceptance_histogram.values()) == sum(r.rounds for r in rep.requests)


@pytest.mark.parametrize("case", [0, 1])
def test_token_sim_under_offload_pressure_matches_reference(case):
    """Token-level serving under KV offload pressure (OFFLOAD policy, small pool): the
    outputs equal the REFERENCE's own run_token_sim outputs for the same workload and pool
    (tests/golden/offload_streams.json, simulate.py:535 run under kvpool.py's offload
    policy), the host tier is physical (bytes left HBM and came back on the copy stream),
    and pages are granted on demand (the device pool is sized to the KvPool capacity)."""
    import json
    from pathlib import Path

    from paper_2512_01278_b200.kvpool import KvPolicy
    gold = json.loads((Path(__file__).parent / "golden" / "offload_streams.json").read_text())[case]
    cfg = M.ModelConfig(2, 4, 2, 8, 48, seed=0)
    kv = KvPoolConfig(capacity_pages=gold["capacity"], page_bytes=64, chunk_pages=16, policy=KvPolicy.OFFLOAD)
    n = gold["n"]
    rep = run_token_sim(_workload(n, gold["input_len"], gold["output_len"], seed=gold["seed"]), cfg,
                        SimConfig(k=3, alpha=0.0, sparsity=0.4, max_batch=n), kv, check_lossless=True)
    assert rep.emitted_tokens == n * gold["output_len"]
    assert {str(r): t for r, t in rep.outputs.items()} == gold["outputs"]
    assert max(r.offloaded_pages for r in rep.iterations) > 0
    off, back = run_token_sim.last_transfer_bytes
    assert off > 0 and back > 0
