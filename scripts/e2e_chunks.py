"""Host-I/O pipeline depth sweep: forward() on pinned host buffers with the
batch cut into sequence ranges (BertEncoderB200.forward_host_packed chunks),
wall-clock per call as bench.py's e2e, plus the device time of the range
graphs replayed back to back (what the chunking costs in compute).

    python scripts/e2e_chunks.py [c2|c3] [chunk specs ...]
"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import harness
    from paper_2210_03052_b200.encoder import BertEncoderB200

    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
    specs = sys.argv[2:] or ["1", "2", "3", "4", "0.3,0.7", "0.2,0.8", "0.2,0.6,0.2", "0.15,0.35,0.35,0.15"]
    bs, mx, preset, layers = {"c2": (16, 256, "bert_base", 12), "c3": (16, 512, "bert_large", 24)}[cfgname]
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config(preset, bs, mx, bt.OptFlags.all_on(), layers=layers)
    w = bt.init_weights(cfg, 0)
    x = torch.from_numpy(harness.gen_input(seqs, cfg.hidden_dim, 0)).pin_memory()
    eng = bt.engine_for(w, cfg)
    big = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    out = torch.empty((bs * mx, cfg.hidden_dim), dtype=torch.float32, pin_memory=True)
    ref = None
    for spec in specs:
        parts = spec.split(",")
        ch = int(parts[0]) if len(parts) == 1 else [float(p) for p in parts]
        bounds = BertEncoderB200.chunk_bounds(seqs.lengths, ch)
        for _ in range(5):
            eng.forward_host_packed(seqs, x, out, chunks=ch)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        same = torch.equal(ref, out)
        ts = []
        for _ in range(30):
            big.zero_()  # L2 flush as bench.py
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.forward_host_packed(seqs, x, out, chunks=ch)
            ts.append(time.perf_counter() - t0)
        # device time of the range graphs back to back
        entries = [eng._graph_entry(bt.SeqLengths(seqs.lengths[b0:b1], mx), cfg, eng._cfg_c) for b0, b1 in bounds]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev = []
        for _ in range(10):
            big.zero_()
            a.record()
            for e in entries:
                e[0].replay()
            b.record()
            torch.cuda.synchronize()
            dev.append(a.elapsed_time(b))
        print(f"{cfgname} chunks {spec:>22}: ranges {[b1 - b0 for b0, b1 in bounds]} e2e mean "
              f"{statistics.mean(ts) * 1e3:.3f} median {statistics.median(ts) * 1e3:.3f} ms | device "
              f"{statistics.median(dev):.3f} ms | bitwise == 1-chunk: {same}", flush=True)


if __name__ == "__main__":
    main()
