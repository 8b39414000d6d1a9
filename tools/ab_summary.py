import json, collections, sys
d = collections.defaultdict(list)
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.jsonl"):
    try:
        r = json.loads(l)
    except Exception:
        print(l.strip()[:300]); continue
    d[(r["linear"], r["M"], r["v"])].append(r["us"])
vs = sorted(set(k[2] for k in d))
for k in sorted(set((k[0], k[1]) for k in d)):
    base = min(d[k + (vs[0],)])
    print(k, "  ".join(f"{v} {min(d[k + (v,)]):7.2f} ({min(d[k + (v,)]) / base:.3f})" for v in vs if d.get(k + (v,))))
