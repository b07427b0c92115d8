"""Summarise ``ncu --set full`` captures of the steady-state forward into the
per-kernel JSON kept under profiles/ (and the per-launch DRAM traffic table
bench.py reports as ``roofline.traffic``).

    python scripts/ncu_summary.py gpurun_out/c2_all_ss.ncu-rep gpurun_out/c3_all_ss.ncu-rep \
        --out profiles/r01_v6_ncu_summary.json --traffic profiles/ncu_traffic.json
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__inst_issued.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active")

# kernel-name prefix -> bench.py kernel-table name, in forward order per layer
ROLES = (("forward_prologue", "prologue"), ("plan_scan", "plan"), ("pack_kernel", "pack"), ("mha_fwd", "mha"), ("gemm_ln_kernel", "gemm_attn_out_ln"),
         ("ln_bias_residual", "ln"), ("unpack_kernel", "unpack"))

_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def _bytes(value: str) -> float:
    num, _, unit = value.partition(" ")
    return float(num.replace(",", "")) * _SCALE.get(unit.strip(), 1)


def read_report(path: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        item = {"report": path.name, "kernel": d.get("Kernel Name", "")[:72]}
        for m in METRICS:
            if m in d:
                item[m] = f"{d[m]} {u.get(m, '')}".strip()
        res.append(item)
    return res


def roles(items: list[dict], tag: str) -> dict:
    """Name each launch by its role in the layer, following the forward's
    order: QKV GEMM, MHA, attn-out GEMM (+ LN0, or the fused GEMM+LN), FFN1
    GEMM, FFN2 GEMM (+ LN1, or the fused GEMM+LN)."""
    named = {}
    nxt = "qkv"  # the next projection of the layer
    for it in items:
        k = it["kernel"]
        traffic = _bytes(it.get("dram__bytes_read.sum", "0 byte")) + _bytes(it.get("dram__bytes_write.sum", "0 byte"))
        name = None
        if k.startswith("void gemm_bf16") or k.startswith("gemm_bf16"):
            name, nxt = {"qkv": ("gemm_qkv", "attn_out"), "attn_out": ("gemm_attn_out", "ffn1"),
                         "ffn1": ("gemm_ffn1_gelu", "ffn2"), "ffn2": ("gemm_ffn2", "qkv")}[nxt]
        elif "gemm_ln_kernel" in k:
            name, nxt = ("gemm_ffn2_ln", "qkv") if nxt == "ffn2" else ("gemm_attn_out_ln", "ffn1")
        else:
            for prefix, role in ROLES:
                if prefix in k:
                    name = role
                    break
            if name == "ln":
                name = "ln0" if nxt == "ffn1" else "ln1"
        if name and f"{tag}:{name}" not in named:
            named[f"{tag}:{name}"] = int(traffic)
    return named


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+", type=Path)
    ap.add_argument("--out", type=Path, required=True)
    ap.add_argument("--traffic", type=Path)
    a = ap.parse_args()
    allitems, traffic = [], {}
    for rep in a.reports:
        items = read_report(rep)
        allitems += items
        traffic.update(roles(items, rep.name.split("_")[0]))
    a.out.write_text(json.dumps(allitems, indent=1) + "\n")
    if a.traffic:
        traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full of the "
                            "steady-state forward (--profile-from-start off, scripts/profile_forward.py, "
                            "scripts/gpu_job_profile.sh); ncu flushes caches between passes, so reads are cold.")
        a.traffic.write_text(json.dumps(traffic, indent=1) + "\n")
    for it in allitems:
        print(f"{it['report'][:10]:10s} {it['kernel'][:50]:50s} {it.get('gpu__time_duration.sum', ''):>14s} "
              f"tensor {it.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', '')}")


if __name__ == "__main__":
    main()
