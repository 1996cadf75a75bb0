#!/usr/bin/env python
"""End-to-end MSA timings on the BASELINE MSA configs (cfg0, cfg2, cfg3, cfg4):
in-memory sequences -> guide tree -> merged MSA rows in host memory, through
the public API (dm.msa on a SeqSet). Prints one JSON line per config with the
tree / align device times, the oracle-equivalent Levenshtein + NW cells and
GCUPS, and (when tests/golden/msa_configs.json has the config) whether the
output hashes equal the reference's.

    python bench_msa.py --configs 0,3,2 [--scale2 1.0] [--scale4 0.1]

wall_s covers the Python API (rows as str objects); api_wall_s the same job
through the C ABI (packed bytes in, one host row buffer out).
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,3,2")
    ap.add_argument("--scale2", type=float, default=1.0)
    ap.add_argument("--scale4", type=float, default=0.1)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--files", action="store_true",
                    help="also time FASTA-to-FASTA (dm.run_align on a FASTA file) and dm.evaluate")
    ap.add_argument("--simulate-world", type=int, default=1,
                    help="run the sharded path with k shards on one GPU (checks, not a speed number)")
    args = ap.parse_args()
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200 import dist as dmdist
    rank, world, local = dmdist.env_rank()
    if world > 1:  # torchrun: one process per GPU, NCCL inside libdmb200
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = dm.Context(local)
    if world > 1:
        dmdist.attach_from_torch(ctx)
    elif args.simulate_world > 1:
        dmdist.simulate_world(ctx, args.simulate_world)
    golden = {}
    gp = os.path.join(ROOT, "tests", "golden", "msa_configs.json")
    if os.path.exists(gp):
        golden = json.load(open(gp))
    for cfg in [int(c) for c in args.configs.split(",")]:
        scale = {2: args.scale2, 4: args.scale4}.get(cfg, 1.0)
        data, offs = dm.synth(cfg, scale)
        seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
        sc = dm.ScoringScheme.protein() if cfg == 3 else dm.ScoringScheme.nucleotide()
        best = None
        api_best = None
        if world == 1:
            # the same job through the C ABI only: packed bytes in, the MSA rows
            # in one host buffer out (no Python str objects)
            import ctypes as C
            from paper_2601_15458_b200._lib import check as _check, dm_stats as _st, lib as _lib
            packed, poffs = dm._pack(seqs)
            for _ in range(args.repeat):
                t0 = time.perf_counter()
                ss = dm.SeqSet(data=packed, offsets=poffs, ctx=ctx)
                h = C.c_void_p()
                st_ = _st()
                _check(_lib().dm_msa(ctx.handle, ss.handle, 42, 100, dm._ptr(sc.table, C.c_int16),
                                     dm._ptr(sc.has_symbol, C.c_uint8), sc.open_surcharge(), sc.gap_extend(),
                                     C.byref(h), C.byref(st_)))
                rows = bytearray(_lib().dm_msa_width(h) * _lib().dm_msa_rows(h))
                _lib().dm_msa_copy_rows(h, (C.c_char * max(len(rows), 1)).from_buffer(rows) if rows else None)
                t = time.perf_counter() - t0
                _lib().dm_msa_free(h)
                del ss
                api_best = t if api_best is None else min(api_best, t)
        for _ in range(args.repeat):
            if world > 1:
                tdist.barrier()
            t0 = time.perf_counter()
            ss = dm.SeqSet(seqs, ctx)
            m = dm.msa(ss, sc, seed=42)
            wall = time.perf_counter() - t0
            if world > 1:  # the job ends when the slowest rank ends
                t = torch.tensor([wall], dtype=torch.float64, device="cuda")
                tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
                wall = float(t[0])
            if best is None or wall < best[0]:
                best = (wall, m)
            del ss
        wall, m = best
        if rank != 0:
            continue
        st = m.stats
        key = f"cfg{cfg}@{scale}"
        match = None
        if key in golden:
            h = hashlib.sha256()
            for r in m.rows:
                h.update(r.encode())
                h.update(b"\n")
            match = h.hexdigest() == golden[key]["rows_sha256"]
        line = {"config": key, "n": len(seqs), "width": m.width, "wall_s": wall, "api_wall_s": api_best,
                "tree_ms": st["tree_ms"], "align_ms": st["align_ms"], "cells": st["cells"],
                "gcups_e2e": st["cells"] / wall / 1e9, "launches": st["launches"], "nw_calls": st["nw_calls"],
                "reference_match": match,
                "reference_cpu_s": (golden[key]["tree_s"] + golden[key]["align_s"]) if key in golden else None,
                "reference_threads": golden[key]["threads"] if key in golden else None,
                "n_gpus": world, "simulated_world": args.simulate_world}
        if args.files and world == 1:
            # FASTA file in -> aligned FASTA file out, and the quality metrics
            import tempfile
            with tempfile.TemporaryDirectory() as d:
                src = os.path.join(d, "in.fa")
                with open(src, "w") as f:
                    for i, s in enumerate(dm.split(data, offs)):
                        f.write(f">s{i}\n{s.decode()}\n")
                kind = "aa" if cfg == 3 else "nt"
                dm.run_align(src, os.path.join(d, "out.fa"), alphabet=kind, ctx=ctx)  # warm
                t0 = time.perf_counter()
                dm.run_align(src, os.path.join(d, "out.fa"), alphabet=kind, ctx=ctx)
                line["fasta_to_fasta_s"] = time.perf_counter() - t0
                line["fasta_out_bytes"] = os.path.getsize(os.path.join(d, "out.fa"))
            t0 = time.perf_counter()
            rep = dm.evaluate(m, seqs, ctx=ctx)
            line["evaluate_s"] = time.perf_counter() - t0
            line["evaluate"] = {k: rep[k] for k in ("pair_count", "p_avg", "distortion", "gap_percent")}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
