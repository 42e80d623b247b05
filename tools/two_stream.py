"""Throughput of two independent compress+decompress pipelines (two codecs, two streams, each
replaying its own CUDA graph of one step) against one pipeline: do the memory-bound kernels
(range, z walk) of one overlap the issue-bound ones (compressor, plane decoder) of the other?"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_12557_b200 import fz, synth
import bench

field, shape, rel, _ = bench.WORKLOADS["c4"]
d = synth.generate(field, shape)
x = torch.from_numpy(d).cuda()
K = 20


def make(stream):
    c = fz.Codec(shape, "cuda")
    out = torch.empty_like(x)
    with torch.cuda.stream(stream):
        c.compress(x, fz.REL, rel, sync=False, stream=stream)
        c.decompress_device(c.out, out=out, stream=stream)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            c.compress(x, fz.REL, rel, sync=False, stream=stream)
            c.decompress_device(c.out, out=out, stream=stream)
    torch.cuda.synchronize()
    return c, out, g


sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
ca, oa, ga = make(sa)
cb, ob, gb = make(sb)
cur = torch.cuda.current_stream()
for n_pipes in (1, 2, 1, 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cur)
    sa.wait_event(e0)
    sb.wait_event(e0)
    for k in range(K):
        g = ga if k % 2 == 0 else gb
        s = sa if (n_pipes == 1 or k % 2 == 0) else sb
        with torch.cuda.stream(s):
            g.replay()
    cur.wait_stream(sa)
    cur.wait_stream(sb)
    e1.record(cur)
    torch.cuda.synchronize()
    print(n_pipes, "pipeline(s):", round(e0.elapsed_time(e1) / K * 1000, 1), "us/step", flush=True)
