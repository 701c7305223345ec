import json, os, sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_04084_b200 as F
import synth
def run(o, i, M, it=20, eager=False):
    cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
    L = F.import_layer(cb, idx, i)
    X = synth.torch_activation(M, i)
    Y = torch.empty((M, o), dtype=torch.float16, device="cuda")
    for _ in range(3):
        F.gemm(L, X, out=Y, algo="expand") if False else F.gemm(L, X, out=Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if eager:
        e0.record()
        for _ in range(it): F.gemm(L, X, out=Y)
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / it
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(it): F.gemm(L, X, out=Y)
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it
os.environ["FASQ_GEMM_TC_DECODE_MAX"] = "0"
for ks in ("", "1", "2", "4", "8"):
    if ks: os.environ["FASQ_GEMM_KSPLIT"] = ks
    elif "FASQ_GEMM_KSPLIT" in os.environ: del os.environ["FASQ_GEMM_KSPLIT"]
    for M in (128, 2048):
        print(json.dumps({"ks": ks or "auto", "M": M, "graph_us": round(run(4096, 4096, M), 2), "eager_us": round(run(4096, 4096, M, eager=True), 2)}), flush=True)
