"""A/B timing of the scene-flow step: per-stage CUDA-event times (median over steps, L2
flushed before each) and the graph-replayed step, for one config and quad count.
Runs against the package of the current working directory (so an older tree can be
timed the same way):  cd <tree> && python /root/repo/tools/sweep_time.py driving 8
"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1801_04720_b200 import SGM, Camera, stack_quads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "driving"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    tag = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(os.getcwd())
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    quads = synth.make_batch(cfg, 0, n, workers=min(n, os.cpu_count() or 1)) \
        if 'workers' in synth.make_batch.__code__.co_varnames else [synth.make_quad(cfg, i) for i in range(n)]
    dev = torch.device("cuda", 0)
    g = SGM.from_config(cfg, max_batch=n)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    out = g.alloc_outputs(n, with_disp=not os.environ.get("SWEEP_NO_DISP"))
    st = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(st):
        for _ in range(3):
            g.scene_flow(imgs, flow, cam, out, stream=st)
        st.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            g.scene_flow(imgs, flow, cam, out, stream=st)
        step = []
        for _ in range(steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            gr.replay()
            e1.record(st)
            e1.synchronize()
            step.append(e0.elapsed_time(e1))
        g.set_timing(True)
        stages = {}
        for _ in range(steps):
            flush.fill_(1)
            g.scene_flow(imgs, flow, cam, out, stream=st)
            st.synchronize()
            for k, v in g.read_timing().items():
                stages.setdefault(k, []).append(v)
    med = {k: round(statistics.median(v), 4) for k, v in stages.items()}
    print(f"{tag} {name}x{n}: step {statistics.median(step):.4f} ms  {med}", flush=True)
    g.close()


if __name__ == "__main__":
    main()
