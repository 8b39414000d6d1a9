"""Turn the raw outputs of tools/gpu_bench_profile.sh (gpurun_out/) into the
tracked evidence under profiles/ (round tag, e.g. r01).

    python tools/summarize_profiles.py r01

Reads gpurun_out/{bench.json, bench_ref.json, bl_all.jsonl, bl_prefill.jsonl,
sweep.jsonl, launches.csv, prof_gate32.ncu-rep, prof_gate1.ncu-rep} and writes
profiles/<tag>_*.{json,jsonl,csv} plus profiles/ncu_summary.json (bench.py
reads `traffic_bytes_per_launch` from it).  Needs `ncu` on PATH for the
.ncu-rep files (it is in this image).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")
TILES = {"gate": 112 * 64, "gateup": 224 * 64}  # 64x128 tiles of 4096x14336 / 4096x28672
ALG = {"gate": 65950928, "gateup": 131910168}  # K*ceil(N/8) + 2*nnz at p=0.5 (seeded bench matrices)


def last_json_line(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith("{")]
    return json.loads(lines[-1])


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def f(v):
    return float(str(v).replace(",", ""))


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    # (a second call may carry only some of the outputs: each part is
    # processed when its file is present)
    if os.path.exists(os.path.join(OUT, "bench.json")):
        b = last_json_line(os.path.join(OUT, "bench.json"))
        json.dump(b, open(os.path.join(PROF, f"{tag}_bench_stack.json"), "w"), indent=1)
    if os.path.exists(os.path.join(OUT, "bench_ref.json")):
        r = last_json_line(os.path.join(OUT, "bench_ref.json"))
        json.dump(r, open(os.path.join(PROF, f"{tag}_bench_reference_arm.json"), "w"), indent=1)
    for src, dst in (("bl_all.jsonl", "per_linear_decode.jsonl"), ("bl_prefill.jsonl", "per_linear_prefill.jsonl"),
                     ("sweep.jsonl", "sweep_4096x14336.jsonl"), ("nm24_perf.jsonl", "nm24_per_linear.jsonl")):
        p = os.path.join(OUT, src)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(PROF, f"{tag}_{dst}"))

    if os.path.exists(os.path.join(OUT, "launches.csv")):
        launch_list(tag)
    ncu_summaries(tag)


def launch_list(tag):
    # launch list: per-launch duration and DRAM bytes of our kernels
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    hdr = next(i for i, row in enumerate(rows) if "Metric Name" in row)
    h = rows[hdr]
    idx = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    launches = {}
    for row in rows[hdr + 1:]:
        if len(row) < len(h):
            continue
        lid = int(row[idx["ID"]])
        d = launches.setdefault(lid, {"id": lid, "kernel": row[idx["Kernel Name"]]})
        name, val = row[idx["Metric Name"]], f(row[idx["Metric Value"]])
        if name == "gpu__time_duration.sum":
            d["us"] = val / 1e3 if val > 1e4 else val  # ns or us depending on ncu units
        elif name.startswith("dram__bytes"):
            d["dram_bytes"] = d.get("dram_bytes", 0.0) + val
    ll = sorted(launches.values(), key=lambda d: d["id"])
    share = {}
    tot = sum(d.get("us", 0.0) for d in ll)
    for d in ll:
        s = share.setdefault(d["kernel"], {"launches": 0, "total_us": 0.0})
        s["launches"] += 1
        s["total_us"] += d.get("us", 0.0)
    for s in share.values():
        s["share"] = s["total_us"] / tot if tot else None
    json.dump({"note": "ncu --metrics gpu__time_duration.sum,dram__bytes_* --clock-control none over "
                       "`bench.py --layers 1` (kernel filter salr_*|adapter_u); per-launch times are cold-cache "
                       "and serialised: compare shares, not absolutes",
               "share_by_kernel": share, "launches": ll},
              open(os.path.join(PROF, f"{tag}_launch_list.json"), "w"), indent=1)



def ncu_summaries(tag):
    # keep earlier captures this run did not redo (e.g. the prefill kernel)
    try:
        summ = {k: v for k, v in json.load(open(os.path.join(PROF, "ncu_summary.json"))).items()
                if isinstance(v, dict)}
    except Exception:
        summ = {}
    logs = {"prof_gateup32": "ncu_fullgu.log", "prof_gate32": "ncu_full.log", "prof_gate1": "ncu_full1.log",
            "prof_prefill_gate2048": "ncu_fullpf.log", "prof_nm24_gate32": "ncu_fullnm.log"}
    for name, shape, tokens in (("prof_gateup32", "gateup", 32), ("prof_gate32", "gate", 32),
                                ("prof_gate1", "gate", 1), ("prof_prefill_gate2048", "gate", 2048),
                                ("prof_nm24_gate32", "gate", 32)):
        alg = ALG[shape]
        try:  # the profiled script prints the matrix's algorithmic bytes
            for line in open(os.path.join(OUT, logs[name])):
                if line.startswith("compressed_bytes"):
                    alg = int(line.split()[1])
        except OSError:
            pass
        rep = os.path.join(OUT, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        recs, units = ncu_raw(rep)
        m = recs[0]
        dur = f(m["gpu__time_duration.sum"])
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = f(m["dram__bytes_read.sum"]) * scale[units["dram__bytes_read.sum"]]
        wr = f(m["dram__bytes_write.sum"]) * scale[units["dram__bytes_write.sum"]]
        summ[name] = {
            "kernel": m["Kernel Name"][:60],
            "shape": shape,
            "tokens": tokens,
            "duration_us_under_ncu": dur,
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "traffic_bytes_per_launch": rd + wr,
            "algorithmic_compressed_bytes": alg,
            "smem_lsu_wavefronts_per_tile": f(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]) / TILES[shape],
            "warp_instructions_per_tile": f(m["smsp__inst_executed.sum"]) / TILES[shape],
            "dram_throughput_pct": f(m.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
            "issue_active_pct": f(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", "nan")),
            "ipc_active": f(m["sm__inst_executed.avg.per_cycle_active"]),
            "tensor_pipe_pct_elapsed": f(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]),
            "note": "ncu --set full --clock-control none, cold cache, serialized",
        }
        with open(os.path.join(PROF, f"{tag}_ncu_{name}_details.csv"), "w") as fo:
            fo.write(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                                    text=True).stdout)
    if "prof_gateup32" in summ:  # the bench's dominant launch (bench.py reads these three keys)
        summ["launch"] = "gateup M=32"
        summ["traffic_bytes_per_launch"] = summ["prof_gateup32"]["traffic_bytes_per_launch"]
        summ["source"] = (f"profiles/{tag}_ncu_prof_gateup32_details.csv: ncu --set full --clock-control none of "
                          "one salr_linear_kernel launch of the bench's gate|up linear (4096x28672, M=32), "
                          "dram__bytes_read.sum + dram__bytes_write.sum")
    json.dump(summ, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in summ.items() if k != "traffic_bytes_per_launch"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
