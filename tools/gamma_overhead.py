"""Per-kernel cost of the resized step vs gamma on one simulated TP rank
(diagnostics for the recovery simulation: what a small gamma costs).

Run under ncu (launch list):
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ztp --csv \
      --log-file gpurun_out/gov.csv python tools/gamma_overhead.py
then  python tools/gamma_overhead.py --parse gpurun_out/gov.csv gpurun_out/gov.json
CFG (c4), TP (8), GAMMAS (0,0.03,0.25,0.5,0.75) from the environment.  Each
gamma runs 3 un-captured steps; the third step's launches are reported."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFG = os.environ.get("CFG", "c4")
TP = int(os.environ.get("TP", "8"))
GAMMAS = [float(x) for x in os.environ.get("GAMMAS", "0,0.03,0.25,0.5,0.75").split(",")]
STEPS = 3


def run():
    import numpy as np
    import torch
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.layer import ZtpLayer, layer_prune_counts
    from synth.configs import CONFIGS
    import bench
    cfg = CONFIGS[CFG]
    h, f, N, e = cfg.h, cfg.f, cfg.N, TP
    a, u = h // e, f // e
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    sh = bench.rank_shards(cfg, e, 0)
    dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
    L = ZtpLayer(ctx, h, f, N, 0, e, dev)
    L.X.normal_()
    L.G.normal_()
    sc = {s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, 0, {"qkv": h, "o": a, "fc1": h, "fc2": u}).items()}
    stream = torch.cuda.Stream()
    meta = []
    for g in GAMMAS:
        p = Z.PlanT()
        p.world = e
        p.role[0] = Z.RESIZE if g > 0 else Z.NORMAL
        p.gamma[0] = p.gamma_r[0] = g
        L.set_selection(layer_prune_counts(p, 0, h, a, u), sc, stream)
        torch.cuda.synchronize()
        n0 = Z.ztp_launch_count(ctx)
        per = []
        for _ in range(STEPS):
            k0 = Z.ztp_launch_count(ctx)
            L.step(stream)
            per.append(Z.ztp_launch_count(ctx) - k0)
        torch.cuda.synchronize()
        meta.append({"gamma": g, "launches_before": n0, "per_step": per, "nk": dict(L.nk)})
    json.dump({"cfg": CFG, "tp": TP, "meta": meta}, open(f"gpurun_out/gov_meta_{CFG}_{TP}.json", "w"), indent=1)
    Z.ztp_ctx_destroy(ctx)


def parse(csv_path, out_path):
    meta = json.load(open(f"gpurun_out/gov_meta_{CFG}_{TP}.json"))
    rows = [r for r in csv.DictReader(l for l in open(csv_path) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    names = [(r["Kernel Name"], float(r["Metric Value"]) / (1e3 if r["Metric Unit"] in ("nsecond", "ns") else 1.0))
             for r in rows]
    # ncu counts select/launch order exactly as ztp_launch_count (one ztp kernel per count)
    idx = 0
    out = []
    for m in meta["meta"]:
        start = m["launches_before"] + sum(m["per_step"][:-1])     # ncu index == library launch count
        n = m["per_step"][-1]
        ks = names[start:start + n]
        out.append({"gamma": m["gamma"], "nk": m["nk"], "total_us": sum(t for _, t in ks),
                    "kernels": [(k.split("(")[0][:60], round(t, 2)) for k, t in ks]})
        idx = start + n
    json.dump(out, open(out_path, "w"), indent=1)
    for o in out:
        print(f"gamma {o['gamma']:.3f}  sum {o['total_us']:.1f} us  nk {o['nk']}")
        for k, t in o["kernels"]:
            print(f"   {t:8.2f}  {k}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--parse":
        parse(sys.argv[2], sys.argv[3])
    else:
        run()
