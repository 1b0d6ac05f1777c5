"""Tabulate trace_serve JSON lines."""
import json, sys
for path in sys.argv[1:]:
    for l in open(path):
        d = json.loads(l)
        m = f"{d['design']} {d['machines']['prompt']}P/{d['machines']['token']}T"
        t = d["trace"]
        if not d.get("sustainable", True):
            print(f"{d['model']:10s} {m:20s} {t['preset']:12s} rate {t['rate']:5.1f} n={t['requests']:4d}  NOT SUSTAINABLE: {d['reason'][:80]}")
            continue
        s = d["summary"]
        print(f"{d['model']:10s} {m:20s} {t['preset']:12s} rate {t['rate']:5.1f} n={t['requests']:4d}  "
              f"TTFT p50 {s['ttft_ms_p50']:7.1f} p99 {s['ttft_ms_p99']:8.1f}  TBT p50 {s['tbt_ms_p50']:6.2f} "
              f"p99 {s['tbt_ms_p99']:7.2f}  E2E p50 {s['e2e_ms_p50']:7.0f}  tok/s {s['tokens_per_s']:6.0f}  "
              f"xfer vis {d['kv_transfer']['visible_ms_p50'] or 0:.2f} raw {d['kv_transfer']['raw_ms_p50'] or 0:.2f} ms  "
              f"dec B {d['iterations']['decode_batch_mean']:.1f}")
