"""forward_host_stream's schedule at C5 re-enacted with events on every copy
and replay: when does each H2D / graph / D2H start and end (ms from t0)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import harness, _lib
    bs, mx, k = 2048, 512, 1024
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    cfg = bt.ModelConfig(layers=24, head_num=16, head_size=64, max_seq_len=mx, batch_size=bs, flags=bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    xh = harness.gen_input(seqs, k, 0)
    x = torch.from_numpy(xh).pin_memory()
    outs = [torch.empty((bs * mx, k), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    eng = bt.engine_for(w, cfg)
    ents = [eng._graph_entry(seqs, cfg, eng._cfg_c, slot=s) for s in range(2)]
    lh = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    K = 4
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = E()
    t0.record()
    for st in (h2d, comp, d2h):
        st.wait_event(t0)
    rec = []
    done, outev = [], []
    for i in range(K):
        e = ents[i % 2]
        a, b, c, d, f, g = E(), E(), E(), E(), E(), E()
        if i >= 2:
            h2d.wait_event(done[i - 2])
        with torch.cuda.stream(h2d):
            a.record()
            _lib.call("bt_copy_rows", e[2].data_ptr(), x.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 1, _lib.stream_ptr())
            b.record()
        comp.wait_event(b)
        if i >= 2:
            comp.wait_event(outev[i - 2])
        with torch.cuda.stream(comp):
            c.record()
            e[0].replay()
            d.record()
        done.append(d)
        d2h.wait_event(d)
        with torch.cuda.stream(d2h):
            f.record()
            _lib.call("bt_copy_rows", outs[i % 2].data_ptr(), e[3].data_ptr(), lh.ctypes.data, bs, mx, k * 4, 0, _lib.stream_ptr())
            g.record()
        outev.append(g)
        rec.append((a, b, c, d, f, g))
    torch.cuda.synchronize()
    for i, (a, b, c, d, f, g) in enumerate(rec):
        print(f"batch {i}: H2D {t0.elapsed_time(a):7.1f}-{t0.elapsed_time(b):7.1f}  graph {t0.elapsed_time(c):7.1f}-"
              f"{t0.elapsed_time(d):7.1f}  D2H {t0.elapsed_time(f):7.1f}-{t0.elapsed_time(g):7.1f}")


if __name__ == "__main__":
    main()
