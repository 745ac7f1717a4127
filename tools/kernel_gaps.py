"""Device idle time inside configs[1] iterations (diagnostics).

Same setup as tools/gpu_only_step.py; then a few eager iterations under torch.profiler
(CUPTI kernel records: start / end / stream).  Prints per iteration the span, the time at
least one kernel is running (union over streams), the idle gaps between kernels, and the
busiest kernels by total time.
    python tools/kernel_gaps.py [--batch 128] [--context 4608] [--iters 3]
"""
import argparse, collections, json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_01278_b200 as sd
from paper_2512_01278_b200 import serving
from paper_2512_01278_b200.engine import DecodeRequest
from paper_2512_01278_b200.scheduler import BatchCandidate, PhaseBuckets, PipelineMode, assign_new_request, first_round_draft_len, form_batch
from paper_2512_01278_b200.workload import synthetic_prompt

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--context", type=int, default=4608)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/kernel_gaps.json")
args = ap.parse_args()
dev = torch.device("cuda")
sd._native.load_library()
cfg = sd.ModelConfig(36, 32, 8, 128, 151936, seed=0)
model = sd.init_model(cfg, dtype=torch.bfloat16, device=dev, fast_init=True)
k, s, B, P = 4, 0.05, args.batch, 512
max_seq = P + 8192
dec = serving.BatchedDecoder(model, k, s, max_requests=B, max_seq_len=max_seq)
reqs = [DecodeRequest(i, synthetic_prompt(0, i, P, cfg.vocab_size) + synthetic_prompt(1, i, args.context - P, cfg.vocab_size),
                      max_seq - args.context) for i in range(B)]
dec.prefill(reqs, max_rows=32768)
bk = PhaseBuckets.empty(k)
for sq in dec.seqs.values():
    sq.round_target = first_round_draft_len(k, assign_new_request(bk))


def it():
    cands = [BatchCandidate(sq.request_id, due_verify=sq.phase == sq.round_target, verify_tokens=sq.round_target + 1)
             for sq in dec.seqs.values() if not sq.done]
    batch, _ = form_batch(cands, [], PipelineMode.SYNCHRONOUS)
    return dec.step(batch.draft_members, batch.verify_members)


for _ in range(10):
    it()
torch.cuda.synchronize()
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(args.iters):
        with torch.profiler.record_function("iteration"):
            it()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
tr = json.load(open(path))
kern = [e for e in tr["traceEvents"] if e.get("cat") == "kernel" and e.get("ph") == "X"]
kern.sort(key=lambda e: e["ts"])
t0, t1 = kern[0]["ts"], max(e["ts"] + e["dur"] for e in kern)
# union of busy intervals and the gaps between them
busy, gaps, cur_s, cur_e = 0.0, [], kern[0]["ts"], kern[0]["ts"] + kern[0]["dur"]
for e in kern[1:]:
    s_, e_ = e["ts"], e["ts"] + e["dur"]
    if s_ > cur_e:
        busy += cur_e - cur_s
        gaps.append((s_ - cur_e, e["name"][:60]))
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
busy += cur_e - cur_s
span = t1 - t0
tot = collections.Counter()
cnt = collections.Counter()
for e in kern:
    nm = e["name"].split("(")[0][:70]
    tot[nm] += e["dur"]
    cnt[nm] += 1
after = collections.Counter()
for g, nm in gaps:
    after[nm.split("(")[0][:50]] += g
res = {"iters": args.iters, "kernels": len(kern), "span_us": span, "busy_us": busy, "idle_us": span - busy,
       "idle_frac": (span - busy) / span, "n_gaps": len(gaps),
       "gap_us_hist": {b: sum(1 for g, _ in gaps if lo <= g < hi) for b, (lo, hi) in
                       {"<1": (0, 1), "1-2": (1, 2), "2-5": (2, 5), "5-20": (5, 20), ">=20": (20, 1e12)}.items()},
       "idle_before": after.most_common(8),
       "top": [(nm, round(t, 1), cnt[nm]) for nm, t in tot.most_common(14)],
       "streams": sorted({e["args"].get("stream") for e in kern})}
print(json.dumps(res, indent=1))
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(res, open(args.out, "w"), indent=1)
L = sd._native.load_library()
print("graph instantiations", L.sd_forward_graph_stats(0), "updates", L.sd_forward_graph_stats(1))
