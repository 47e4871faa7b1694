"""Small-shape probe: where do the paper-sweep shapes that trail cuBLASLt lose their time?

Per shape, times ours and cuBLASLt's fused bias+ReLU (torch._addmm_activation) three ways:
  graph1  one CUDA graph per call, replayed back to back (the paper_sweep.py protocol: includes the
          per-graph launch gap)
  graphN  one CUDA graph holding R calls over rotating operand sets (launch gaps amortised; PDL lets
          our prologue overlap the previous call's tail)
  eager   R eager calls from Python
usage: python scripts/small_probe.py [--r 40]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_12645_b200 as ge  # noqa: E402

SHAPES = [(1152, 256, 128), (512, 128, 512), (640, 2048, 1408), (896, 1408, 1920), (768, 1024, 3456),
          (256, 4096, 2944), (1664, 896, 896), (1408, 1536, 256), (1536, 1280, 2432), (4096, 512, 1536),
          (2048, 2048, 2048)]


def t_graph1(fn, nsets, it=40):
    gs = []
    for i in range(nsets):
        fn(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(i)
        gs.append(g)
    for g in gs:
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(it):
        gs[i % nsets].replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


def t_graphN(fn, nsets, r):
    for i in range(nsets):
        fn(i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(r):
            fn(i % nsets)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * r) * 1e3


def t_eager(fn, nsets, r):
    for i in range(nsets):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(r):
        fn(i % nsets)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / r * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=40)
    ap.add_argument("--ncu", action="store_true", help="3 eager calls per shape and impl only (for an ncu launch list)")
    a = ap.parse_args()
    torch.manual_seed(0)
    for (M, N, K) in SHAPES:
        nsets = max(1, min(8, int(3 * 126e6 // (2 * (M * K + K * N))) + 1))
        sets = [(torch.randn(M, K, device="cuda", dtype=torch.float16) * 0.5,
                 torch.randn(N, K, device="cuda", dtype=torch.float16).t() * 0.5) for _ in range(nsets)]
        bias = torch.randn(N, device="cuda", dtype=torch.float16)
        C = torch.empty(M, N, device="cuda", dtype=torch.float16)
        ours = lambda i: ge.gemm_epilogue(sets[i][0], sets[i][1], bias, out=C)  # noqa: E731
        lt = lambda i: torch._addmm_activation(bias, sets[i][0], sets[i][1])  # noqa: E731
        if a.ncu:
            for fn in (ours, lt):
                for i in range(3):
                    fn(i % nsets)
            torch.cuda.synchronize()
            continue
        row = {"M": M, "N": N, "K": K, "plan": ge.plan(M, N, K, layouts="rc")}
        for name, fn in (("ours", ours), ("lt", lt)):
            row[name] = {"graph1_us": round(t_graph1(fn, nsets), 2), "graphN_us": round(t_graphN(fn, nsets, a.r), 2),
                         "eager_us": round(t_eager(fn, nsets, a.r), 2)}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
