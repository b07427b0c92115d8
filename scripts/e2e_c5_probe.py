"""C5 host-I/O components: pinned output allocation, host zeroing of the
padded rows, valid-row H2D / D2H, and the per-call / stream forwards."""
import sys, time, statistics
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
    x = torch.from_numpy(harness.gen_input(seqs, k, 0)).pin_memory()
    eng = bt.engine_for(w, cfg)
    y = bt.forward(w, seqs, x, cfg)
    torch.cuda.synchronize()
    def wall(fn, n=3):
        ts = []
        for _ in range(n):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3
    print(f"torch.empty pinned 4.3 GB: {wall(lambda: torch.empty((bs * mx, k), dtype=torch.float32, pin_memory=True)):.1f} ms")
    out = torch.empty((bs * mx, k), dtype=torch.float32, pin_memory=True)
    o = out.numpy().reshape(bs, mx, k)
    def zero():
        for b, n in enumerate(seqs.lengths):
            if n < mx:
                o[b, n:] = 0.0
    print(f"host zeroing of padded rows: {wall(zero):.1f} ms")
    graph, run, xp, yp, _, _ = eng._graph_entry(seqs, cfg, eng._cfg_c)
    lh = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
    print(f"H2D valid rows: {wall(lambda: _lib.call('bt_copy_rows', xp.data_ptr(), x.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 1, _lib.stream_ptr())):.1f} ms")
    print(f"D2H valid rows: {wall(lambda: _lib.call('bt_copy_rows', out.data_ptr(), yp.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 0, _lib.stream_ptr())):.1f} ms")
    print(f"graph replay: {wall(lambda: graph.replay()):.1f} ms")
    print(f"forward_host_packed: {wall(lambda: eng.forward_host_packed(seqs, x, out)):.1f} ms")
    print(f"forward(): {wall(lambda: bt.forward(w, seqs, x, cfg)):.1f} ms")


if __name__ == "__main__":
    main()
