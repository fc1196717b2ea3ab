"""Print the headline numbers of bench JSON lines (dev helper)."""
import json
import sys

for f in sys.argv[1:]:
    d = json.load(open(f))
    print(f, "value", round(d["value"]), "ms/step", round(d["ms_per_step"], 4), "clk", (d.get("clocks") or {}).get("sm_mhz"))
    for k, r in d["per_config"].items():
        rf = r["roofline"]
        print(f"  {k}: {r['ms_per_step']:.4f} ms/step {r['gflops']:.0f} GFLOP/s  roof[{rf['bound']} {rf['kernel'][:22]}] "
              f"frac {rf['frac']:.3f} ({rf['achieved']:.1f}/{rf['peak']:.1f} {rf['unit']})")
        for nv, p in r["per_nv"].items():
            ph = {a: round(b, 3) for a, b in p["phases_ms"].items() if b > 0.003}
            print(f"    nv={nv}: {p['ms_per_matvec']:.4f} ms {p['gflops']:.0f} GF/s path {p['path_frac_of_hbm']:.3f} {ph}")
        if r.get("latency_us"):
            print("    latency", r["latency_us"])
