"""Why planted alpha < 1 in bf16 (diagnostics).

In the reference's fp64 planted model every non-planted logit gets +0 against +2000 on
the planted positions, so drafts (critical set covers the planted positions) and verify
see the same attention and alpha = 1 by construction.  In bf16 the draft row and the
verify row of the same token run through different kernels (K1 head-packed vs K2
clusters) and GEMMs of different batch sizes (cuBLAS picks per-M kernels), so their
logits differ by bf16-rounding noise.  This tool runs the configs[1]-shaped planted model
through BatchedDecoder and, for every rejected draft, prints the verify row's margin
between its argmax and the drafted token, and the draft row's margin between the drafted
token and the verify's choice: rejections with both margins inside the noise are
near-ties that bf16 arithmetic cannot order consistently, not kernel errors.

    python tools/alpha_margin.py [--requests 16] [--steps 40]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2512_01278_b200 as sd
from paper_2512_01278_b200.engine import DecodeRequest
from paper_2512_01278_b200.scheduler import BatchCandidate, PipelineMode, form_batch
from paper_2512_01278_b200.serving import BatchedDecoder
from paper_2512_01278_b200.workload import synthetic_prompt

ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=16)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--ctx", type=int, default=1024)
args = ap.parse_args()
dev = torch.device("cuda")
cfg = sd.ModelConfig(36, 32, 8, 128, 151936, seed=0)
model = sd.init_model(cfg, dtype=torch.bfloat16, device=dev, fast_init=True)
model = sd.plant_attention_concentration(model, list(range(5, 512, 512 // 12))[:12])
dec = BatchedDecoder(model, 4, 0.05, max_requests=args.requests, max_seq_len=args.ctx + 512)
reqs = [DecodeRequest(r, synthetic_prompt(0, r, 512, cfg.vocab_size) + synthetic_prompt(1, r, args.ctx - 512,
                                                                                        cfg.vocab_size), 400)
        for r in range(args.requests)]
dec.prefill(reqs)
dec.keep_logits = True
draft_rows = {}   # request -> {phase: logits row}
rej, acc_n = [], 0
for _ in range(args.steps):
    cands = [BatchCandidate(s.request_id, due_verify=s.phase == s.round_target, verify_tokens=s.round_target + 1)
             for s in dec.seqs.values() if not s.done]
    batch, _ = form_batch(cands, [], PipelineMode.SYNCHRONOUS)
    phases = {r: dec.seqs[r].phase for r in batch.draft_members}
    verify_rows = {}
    row = len(batch.draft_members)
    for r in batch.verify_members:
        verify_rows[r] = (row, dec.seqs[r].round_target + 1)
        row += dec.seqs[r].round_target + 1
    res = dec.step(batch.draft_members, batch.verify_members)
    lg = dec.last_logits
    for i, r in enumerate(batch.draft_members):
        draft_rows.setdefault(r, {})[phases[r]] = lg[i].float().clone()
    for r, (row0, t) in verify_rows.items():
        s = dec.seqs[r]
        a = res.accepted[r]
        rec = s.stats.rounds[-1]
        acc_n += a
        if a < t - 1:
            vrow = lg[row0 + a].float()
            target = int(vrow.argmax())
            drow = draft_rows.get(r, {}).get(a)
            drafted = int(drow.argmax()) if drow is not None else -1
            m_verify = float(vrow[target] - vrow[drafted]) if drafted >= 0 else float("nan")
            m_draft = float(drow[drafted] - drow[target]) if drow is not None else float("nan")
            rej.append((m_verify, m_draft, float(vrow.abs().max())))
        draft_rows.pop(r, None)
rej = np.array(rej) if rej else np.zeros((0, 3))
print(json.dumps({"rejections": len(rej), "accepted_drafts": acc_n,
                  "verify_margin": {"median": float(np.median(rej[:, 0])) if len(rej) else None,
                                    "p90": float(np.percentile(rej[:, 0], 90)) if len(rej) else None,
                                    "max": float(rej[:, 0].max()) if len(rej) else None},
                  "draft_margin": {"median": float(np.median(rej[:, 1])) if len(rej) else None,
                                   "p90": float(np.percentile(rej[:, 1], 90)) if len(rej) else None,
                                   "max": float(rej[:, 1].max()) if len(rej) else None},
                  "logit_scale_max": float(rej[:, 2].max()) if len(rej) else None}))
