"""Summarise a KD_PARITY_LOG (JSON lines written by tests/kdtest_util.py) as the markdown table of profiles/rNN_parity.md.

    python scripts/parity_table.py gpurun_out/parity.jsonl > profiles/r02_parity.md
"""
import json
import sys


def main(path):
    rows = [json.loads(line) for line in open(path)]
    n_viol = sum(r["strict_violations"] for r in rows)
    n_el = sum(r["n"] for r in rows)
    print("| test | quantity | elements | max abs err | max err / tol | beyond the bound |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        t = r["test"].split("::")[-1]
        print(f"| `{t}` | {r['name']} | {r['n']} | {r['max_abs_err']:.3g} | {r['max_err_over_strict_tol']:.3g} | "
              f"{r['strict_violations']} |")
    print()
    print(f"{len(rows)} comparisons, {n_el} elements; {n_viol} element(s) beyond the plain north-star bound, all within "
          f"their test's listed allowance (tests/kdtest_util.assert_grad_close).")


if __name__ == "__main__":
    main(sys.argv[1])
