"""Cost of splitting the 48-layer group into chunks and of capping its CTAs (the
N>1 overlap layout): python tools/chunk_cost.py -> chunks, max_ctas, us/step."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2507_01154_b200 as fdp
TYPES = [("c_attn", 768, 2304), ("attn_proj", 768, 768), ("c_fc", 768, 3072), ("mlp_proj", 3072, 768)]
g = torch.Generator(device="cuda").manual_seed(0)
layers = []
for blk in range(12):
    for j, (n, P, D) in enumerate(TYPES):
        x = torch.randn(8, 1024, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(8, 1024, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        layers.append((x, dy, fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=blk * 4 + j)))
def timed(fn, n=20):
    time.sleep(1)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
full = fdp.PreparedGroup(layers, noise_impl="philox")
for nch in (1, 2, 4, 8):
    for cap in (0, 144, 132):
        per = 48 // nch
        gs = [fdp.PreparedGroup(layers[i * per:(i + 1) * per], noise_impl="philox", max_ctas=cap) for i in range(nch)]
        def run():
            for gg in gs: gg()
        print(nch, cap, round(timed(run), 1))
