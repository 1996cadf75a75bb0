#!/usr/bin/env python
"""Where the end-to-end MSA wall time goes outside the kernels (cfg4 by default)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200._lib import check, lib, dm_stats
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    data, offs = dm.synth(cfg, 1.0)
    seqs = list(dict.fromkeys(s.decode() for s in dm.split(data, offs)))
    ctx = dm.default_context(0)
    sc = dm.ScoringScheme.nucleotide()
    for rep in range(2):
        t0 = time.perf_counter()
        ss = dm.SeqSet(seqs, ctx)
        t1 = time.perf_counter()
        h = C.c_void_p()
        s = dm_stats()
        check(lib().dm_msa(ctx.handle, ss.handle, 42, 100, dm._ptr(sc.table, C.c_int16), dm._ptr(sc.has_symbol, C.c_uint8),
                           sc.open_surcharge(), sc.gap_extend(), C.byref(h), C.byref(s)))
        t2 = time.perf_counter()
        m = dm._msa_from(h)
        lib().dm_msa_free(h)
        t3 = time.perf_counter()
        print(f"rep {rep}: seqset {1e3*(t1-t0):.1f} ms, dm_msa {1e3*(t2-t1):.1f} ms (tree {s.tree_ms:.1f} + align "
              f"{s.align_ms:.1f}), to python {1e3*(t3-t2):.1f} ms, width {m.width}")


if __name__ == "__main__":
    main()
