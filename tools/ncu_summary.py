"""Summarise an ncu report (+ optional launch-list CSV) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [gpurun_out/launches.csv] --tag r1a \
        [--traffic-json profiles/ncu_traffic.json] [--emt-steps 200 --lanes 1000 --bytes-per 8848]
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--traffic-json")
    ap.add_argument("--emt-steps", type=int, default=0)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--bytes-per", type=int, default=0)
    a = ap.parse_args()
    head, units, rows = raw(a.rep)
    summ = {"report": os.path.basename(a.rep), "kernels": []}
    for r in rows:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        k = {"name": d.get("Kernel Name", "")[:80]}
        for key in KEYS:
            if key in d:
                k[key] = f"{d[key]} {u.get(key, '')}".strip()
        stalls = []
        for i, key in enumerate(head):
            if "pcsamp_warps_issue_stalled" in key and not key.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), key.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        k["stall_share"] = {name: round(x / tot, 3) for x, name in sorted(stalls, reverse=True)[:8]}
        summ["kernels"].append(k)
    if a.launches and os.path.exists(a.launches):
        lines = [l for l in open(a.launches) if l.startswith('"ID"') or l[:2] == '"0' or l[:1] == '"']
        rdr = csv.reader(io.StringIO("".join(lines)))
        hdr = next(rdr)
        launches = []
        for r in rdr:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                launches.append((d.get("Kernel Name", "")[:60], d.get("Metric Unit"), float(d["Metric Value"].replace(",", ""))))
        tot = {}
        for name, unit, v in launches:
            tot.setdefault(name, [0.0, 0, unit])
            tot[name][0] += v
            tot[name][1] += 1
        all_t = sum(v[0] for v in tot.values()) or 1.0
        summ["launch_list"] = {n: {"launches": c, "total": t, "unit": u, "share": round(t / all_t, 4)}
                               for n, (t, c, u) in tot.items()}
    os.makedirs("profiles", exist_ok=True)
    out = os.path.join("profiles", f"ncu_{a.tag}.json")
    json.dump(summ, open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1))
    if a.traffic_json and summ["kernels"]:
        k = summ["kernels"][0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def nbytes(v):
            num, unit = (v.split() + ["byte"])[:2]
            return float(num) * scale.get(unit, 1)

        traffic = nbytes(k["dram__bytes_read.sum"]) + nbytes(k["dram__bytes_write.sum"])
        info = {"dram_bytes_per_launch": traffic, "source": out, "kernel": k["name"],
                "emt_steps_per_launch": a.emt_steps, "lanes": a.lanes}
        if a.emt_steps:
            info["dram_bytes_per_emt_step"] = traffic / a.emt_steps
        if a.bytes_per and a.emt_steps and a.lanes:
            info["algorithmic_bytes_per_launch"] = a.bytes_per * a.emt_steps * a.lanes
        json.dump(info, open(a.traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main()
