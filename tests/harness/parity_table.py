"""Markdown table of a run_configs.py --certify --oracle JSONL (one row per
(config, ω)): python tests/harness/parity_table.py IN.jsonl > OUT.md-fragment"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("| config | ω | oracle ω | phases | status | sweeps | GPU time-to-ε | z_rel | P_rel | D_rel "
      "| cert (oracle) | oracle time |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
f = lambda x: "—" if x is None else f"{x:.2e}"
for r in rows:
    ok = r["status"] == 0
    print(f"| {r['name']} | {r['omega']} | {r.get('oracle_omega', '—')} | {r['colors']} | {r['status']} "
          f"| {r['sweeps']} | {r['solve_ms']:.1f} ms | {f(r.get('z_rel_vs_oracle')) if ok else '—'} "
          f"| {f(r.get('P_rel_vs_oracle')) if ok else '—'} | {f(r.get('D_rel_vs_oracle')) if ok else '—'} "
          f"| {r['oracle_cert_ratio']:.4f} | {r.get('oracle_s', 0):.1f} s |" if ok else
          f"| {r['name']} | {r['omega']} | — | {r['colors']} | {r['status']} | {r['sweeps']} "
          f"| {r['solve_ms']:.1f} ms | — | — | — | — | — |")
