"""How does compute time depend on batch chunking? (debug)"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1801_04720_b200 import SGM, Camera, stack_quads
cfg = synth.CONFIGS["batch"]; prm = synth.sgm_params(cfg)
cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
dev = torch.device("cuda")
quads = [synth.make_quad(cfg, i) for i in range(8)]
g8 = SGM.from_config(cfg, max_batch=8)
imgs, flow = stack_quads(quads, g8.pitch, dev)
out8 = g8.alloc_outputs(8)
gs = [SGM.from_config(cfg, max_batch=4) for _ in range(4)]
outs = [g.alloc_outputs(4) for g in gs]
streams = [torch.cuda.Stream() for _ in range(4)]
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
def one8(): g8.scene_flow(imgs, flow, cam, out8)
def chunks(nstreams, cq=2):
    def f():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event(); ev.record(cur)
        for c in range(8 // cq):
            s = streams[c % nstreams]; s.wait_event(ev)
            o = {k: v[:cq] for k, v in outs[c].items()}
            gs[c].scene_flow(imgs[cq*c:cq*c+cq], flow[cq*c:cq*c+cq], cam, o, stream=s)
        for c in range(nstreams):
            cur.wait_stream(streams[c])
    return f
print("8 quads, 1 launch set: %.2f ms" % t(one8))
print("4 x 2 quads, 1 stream: %.2f ms" % t(chunks(1)))
print("4 x 2 quads, 2 streams: %.2f ms" % t(chunks(2)))
print("4 x 2 quads, 4 streams: %.2f ms" % t(chunks(4)))
g1 = SGM.from_config(cfg, max_batch=1); o1 = g1.alloc_outputs(1)
print("2 x 4 quads, 2 streams: %.2f ms" % t(chunks(2, 4)))
print("[3,3,2] n/a; 1 quad latency: %.2f ms" % t(lambda: g1.scene_flow(imgs[:1], flow[:1], cam, o1)))
