"""Summarise bench JSON lines (one file per config) as the markdown table of profiles/rNN_bench_final.md.

    python scripts/bench_table.py gpurun_out/final/{default,c3_rkl,c3_jsd,c4,c5}.jsonl
"""
import json
import os
import sys


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(f"no JSON line in {path}")


def main(paths):
    print("| config | tokens/s (median step) | ms/step | e2e tokens/s | dominant kernel | roofline frac (sustained) "
          "| SM MHz | power W | tokens/J |")
    print("|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        d = last_json(p)
        r, c, e = d["roofline"], d["clocks"], d.get("energy") or {}
        name = os.path.basename(p).split(".")[0]
        e2e = d["e2e"]["value"] if isinstance(d.get("e2e"), dict) and "value" in d["e2e"] else None
        print(f"| {name} | {d['value']:.0f} | {d['ms_per_step']:.2f} | {e2e:.0f} | {r['kernel']} | {r['frac']:.3f} | "
              f"{c.get('sm_mhz')} | {c.get('power_w_median')} | {e.get('tokens_per_joule', float('nan')):.1f} |"
              if e2e is not None else
              f"| {name} | {d['value']:.0f} | {d['ms_per_step']:.2f} | — | {r['kernel']} | {r['frac']:.3f} | "
              f"{c.get('sm_mhz')} | {c.get('power_w_median')} | {e.get('tokens_per_joule', float('nan')):.1f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
