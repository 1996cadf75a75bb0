#!/usr/bin/env python
"""HBM evidence for the memory-bound passes around the DP kernels (SURVEY.md
§8(d), VERDICT r1 "what's missing" 6): one FASTA -> aligned FASTA run of a
BASELINE config through dm_run_align, which launches the sequence-set
kernels (census / recode2 / planes), the merge passes (colmap /
insert_rows, the NW traceback) and the FASTA formatter.

  python tools/prof_mem.py --cfg 2 [--scale 1.0]            # plain run, writes the algorithmic-bytes log
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      -k regex:'census|recode|planes|colmap|insert_rows|traceback|fasta_format|init_rows' \\
      --csv --log-file gpurun_out/mem.csv python tools/prof_mem.py --cfg 2
  python tools/prof_mem.py --summarize gpurun_out/mem.csv gpurun_out/mem_bytes.log

The summary lists, per kernel: launches, device time, DRAM bytes (ncu),
algorithmic bytes (the library's DM_TRACE_BYTES log: bytes each launch must
read + write), achieved GB/s of both against MEASURED_PEAKS.json hbm_gbs."""
import argparse
import collections
import csv
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg, scale, log):
    os.environ["DM_TRACE_BYTES"] = "1"
    import paper_2601_15458_b200 as dm
    data, offs = dm.synth(cfg, scale)
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "in.fa")
        with open(src, "w") as f:
            for i, s in enumerate(dm.split(data, offs)):
                f.write(f">s{i}\n{s.decode()}\n")
        fd = os.open(log, os.O_WRONLY | os.O_CREAT | os.O_TRUNC)
        os.dup2(fd, 2)  # the library's byte log goes to stderr
        dm.run_align(src, os.path.join(d, "out.fa"), alphabet="aa" if cfg == 3 else "nt")


def summarize(ncu_csv, bytes_log):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.8
    algo = collections.defaultdict(lambda: [0, 0, 0])
    for line in open(bytes_log):
        if line.startswith("[dm bytes]"):
            _, _, k, r, w = line.split()
            a = algo[k]
            a[0] += 1
            a[1] += int(r)
            a[2] += int(w)
    rows = [r for r in csv.reader(l for l in open(ncu_csv) if not l.startswith("=="))]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        m = r[mi]
        a = agg[name]
        if m == "gpu__time_duration.sum":
            a["n"] += 1
            a["ns"] += v
        elif m == "dram__bytes_read.sum":
            a["rd"] += v
        elif m == "dram__bytes_write.sum":
            a["wr"] += v
    out = []
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        t = a["ns"] * 1e-9
        al = algo.get(name)
        rec = {"kernel": name, "launches": a["n"], "time_ms": a["ns"] * 1e-6,
               "dram_bytes": a["rd"] + a["wr"], "dram_gbs": (a["rd"] + a["wr"]) / t / 1e9 if t else None}
        rec["dram_frac_of_hbm"] = rec["dram_gbs"] / peak if rec["dram_gbs"] else None
        if al and al[0] == a["n"]:
            rec["algorithmic_bytes"] = al[1] + al[2]
            rec["algorithmic_gbs"] = (al[1] + al[2]) / t / 1e9
            rec["algorithmic_frac_of_hbm"] = rec["algorithmic_gbs"] / peak
            rec["dram_over_algorithmic"] = rec["dram_bytes"] / max(1, rec["algorithmic_bytes"])
        out.append(rec)
    for r in out:
        print(json.dumps(r))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--log", default=os.path.join(ROOT, "gpurun_out", "mem_bytes.log"))
    ap.add_argument("--summarize", nargs=2, metavar=("NCU_CSV", "BYTES_LOG"))
    a = ap.parse_args()
    if a.summarize:
        summarize(*a.summarize)
    else:
        os.makedirs(os.path.dirname(a.log), exist_ok=True)
        run(a.cfg, a.scale, a.log)


if __name__ == "__main__":
    main()
