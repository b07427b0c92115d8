"""BASELINE.json configs[3] ("C4"): BERT-base 12-layer sweep, batch 1-64 x
max_seq 64-1024, lengths gen_lengths(fixed, alpha 0.6), padded baseline
(OptFlags(): every kernel over bs*mx rows, padded MHA) vs padding-free
(OptFlags.all_on()), both on the B200 kernels through run_ladder.

    python scripts/sweep_c4.py [--out profiles/r01_c4_sweep.csv] [--repeats 5]
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 8, 16, 32, 64])
    ap.add_argument("--max-lens", type=int, nargs="+", default=[64, 128, 256, 512, 1024])
    a = ap.parse_args()
    from paper_2210_03052_b200.bench_ladder import BenchSpec, run_ladder

    lines = ["batch,max_len,tokens_padded,alpha,padded_ms,padding_free_ms,speedup,padded_seq_per_s,"
             "padding_free_seq_per_s,max_rel_dev"]
    ok = True
    for bs in a.batches:
        for mx in a.max_lens:
            spec = BenchSpec(preset="bert_base", batch_size=bs, max_seq_lens=(mx,), alphas=(0.6,), mode="fixed",
                             repeats=a.repeats, variants=("baseline", "fused_mha"))
            res = run_ladder(spec)
            ok &= res.passed
            r = {row.variant: row for row in res.rows}
            b, f = r["baseline"], r["fused_mha"]
            lines.append(f"{bs},{mx},{bs * mx},{f.alpha_actual:.4f},{b.median_ms:.4f},{f.median_ms:.4f},"
                         f"{b.median_ms / f.median_ms:.3f},{bs / (b.median_ms / 1e3):.1f},"
                         f"{bs / (f.median_ms / 1e3):.1f},{f.max_rel_dev:.3e}")
            print(lines[-1], flush=True)
    text = "\n".join(lines) + "\n"
    if a.out:
        Path(a.out).write_text(text)
    return 0 if ok else 1


if __name__ == "__main__":
    raise SystemExit(main())
