"""Device-only time of one configs[1] unified iteration (diagnostics).

Runs bench.py's setup, then captures one iteration's forward (all 36 layers:
norms, GEMMs, RoPE/KV append, K1 + K2 attention, LM head, argmax) into a CUDA
graph and replays it: the replay time is what the GPU needs without host
launch overhead.  Compare with bench.py's ms_per_step / host.enqueue_ms.
    python tools/gpu_only_step.py [--batch 128] [--context 4608]
"""
import argparse, os, sys, time
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
ap.add_argument("--layers", type=int, default=36)
args = ap.parse_args()
dev = torch.device("cuda")
sd._native.load_library()
cfg = sd.ModelConfig(args.layers, 32, 8, 128, 151936, seed=0)
model = sd.init_model(cfg, dtype=torch.bfloat16, device=dev, fast_init=True)
k, s, B, P = 4, 0.05, args.batch, 512
max_seq = P + 8192
dec = serving.BatchedDecoder(model, k, s, max_requests=B, max_seq_len=max_seq)
reqs = [DecodeRequest(i, synthetic_prompt(0, i, P, cfg.vocab_size) + synthetic_prompt(1, i, args.context - P, cfg.vocab_size),
                      max_seq - args.context) for i in range(B)]
seqs = dec.prefill(reqs, max_rows=32768)
bk = PhaseBuckets.empty(k)
for sq in seqs:
    sq.round_target = first_round_draft_len(k, assign_new_request(bk))

def it():
    cands = [BatchCandidate(sq.request_id, due_verify=sq.phase == sq.round_target, verify_tokens=sq.round_target + 1)
             for sq in dec.seqs.values() if not sq.done]
    batch, _ = form_batch(cands, [], PipelineMode.SYNCHRONOUS)
    return dec.step(batch.draft_members, batch.verify_members)

for _ in range(int(os.environ.get("WARM", "8"))):
    it()
torch.cuda.synchronize()
n0 = len(dec.host_times)
t0 = time.perf_counter()
per = []
for _ in range(10):
    tt = time.perf_counter()
    rr = it()
    per.append((round((time.perf_counter() - tt) * 1e3, 2), rr.draft_rows, rr.verify_rows, round(dec.host_times[-1][0] * 1e3, 2)))
torch.cuda.synchronize()
print("per step (ms, draft rows, verify rows, enqueue ms):", per)
t10 = (time.perf_counter() - t0) / 10
ht = dec.host_times[n0:]
print(f"10 eager steps: {t10 * 1e3:.2f} ms/step, host enqueue {1e3 * sum(a for a, _ in ht) / len(ht):.2f} ms, "
      f"enqueue+drain {1e3 * sum(b for _, b in ht) / len(ht):.2f} ms")
captured = {}
real = serving.forward_rows
def spy(*a, **kw):
    captured["args"], captured["kw"] = a, kw
    return real(*a, **kw)
serving.forward_rows = spy
torch.cuda.synchronize()
t0 = time.perf_counter()
r = it()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
serving.forward_rows = real
a, kw = captured["args"], captured["kw"]
launches = [ln for ln in a[5]]
for ln in launches:
    ln.timer = None
from paper_2512_01278_b200.model import lm_head
def fwd():
    x = real(*a[:5], launches, **kw)
    return serving._argmax(lm_head(model, x))
fwd(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    fwd()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        fwd()
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"rows {r.rows} (draft {r.draft_rows}, verify {r.verify_rows}); eager step wall {wall * 1e3:.2f} ms; "
      f"graph replay of the forward {e0.elapsed_time(e1) / n:.2f} ms; host enqueue {dec.host_times[-1][0] * 1e3:.2f} ms")
