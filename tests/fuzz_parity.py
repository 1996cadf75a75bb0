#!/usr/bin/env python
"""Time-budgeted randomised parity campaign: libdmb200 (GPU) vs the compiled
reference (oracle/_ref) on seeded random inputs and random settings of the
library's kernel-choice knobs. Test infrastructure (the oracle is the checker):

    python tests/fuzz_parity.py --seconds 600 --seed 1 [--kinds lev,nw,...]

Every case is reproducible from (seed, case number); a mismatch prints the
case and the campaign goes on. `tests/test_fuzz_gpu.py` runs a short campaign
under `-m gpu`. What is compared, bit for bit:
  lev      dm_lev_pairs on a resident set        vs divmsa::levenshtein (distance.cpp:9-48)
  packed   dm_lev_pairs_packed from host memory  vs the same
  scan     dm_lev_one_to_many                    vs distance_scan (cluster_tree.cpp:31-41)
  nw       dm_nw_batch                           vs nw_align (pairwise.cpp:301-415)
  tree     dm_build_tree                         vs build_tree (cluster_tree.cpp:168-235)
  msa      dm_msa                                vs build_tree + align_all (msa_merge.cpp:107-158)
  align    dm_align_sequences (duplicates)       vs align_sequences (pipeline.cpp:78-159)
  fasta    dm_run_align: FASTA in, aligned FASTA + tree / dedup dumps out vs run_align (pipeline.cpp:160-187)
  metrics  dm_evaluate                           vs evaluate (metrics.cpp:84-169)
"""
import argparse
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

ALPHABETS = {
    "bin": "AC",
    "dna": "ACGT",
    "dna5": "ACGTN",
    "iupac": "ACGTRYSWKMBDHVN",
    "aa": "ARNDCQEGHILKMFPSTWYV",
    "aa24": "ARNDCQEGHILKMFPSTWYVBZX*",
    "ascii": "".join(chr(c) for c in range(33, 127) if chr(c) not in "->"),
}
KNOBS = ("DM_LEV_GPAR", "DM_LEV_WMAX", "DM_NW_SEQ", "DM_NW_CLU", "DM_TREE_BG", "DM_TREE_CACHE", "DM_NW_TRACE_GB",
         "DM_STREAM_CHUNK_BYTES", "DM_STREAM_PACK", "DM_STREAM_HOSTPLAN", "DM_STREAM_RAW_FRAC")


def rand_len(rng, hi):
    """Lengths that hit the word / band edges as well as the bulk."""
    k = rng.random()
    if k < 0.15:
        return rng.randint(0, 5)
    if k < 0.45:
        edge = rng.choice((32, 64, 96, 128, 256, 384, 512, 1024, 1536, 2048))
        return max(0, min(hi, edge + rng.randint(-2, 2)))
    if k < 0.9:
        return rng.randint(1, max(1, min(hi, 600)))
    return rng.randint(1, hi)


def rand_seq(rng, n, alpha):
    return "".join(rng.choices(alpha, k=n))


def mutate(rng, s, alpha, rate):
    out = []
    for ch in s:
        r = rng.random()
        if r < rate * 0.6:
            out.append(rng.choice(alpha))
        elif r < rate * 0.8:
            continue
        elif r < rate:
            out.append(ch)
            out.append(rng.choice(alpha))
        else:
            out.append(ch)
    return "".join(out)


def rand_set(rng, count, hi, alpha, min_len=0):
    """A mix of unrelated sequences and mutated copies (small distances)."""
    seqs = []
    while len(seqs) < count:
        if seqs and rng.random() < 0.5:
            s = mutate(rng, rng.choice(seqs), alpha, rng.choice((0.01, 0.05, 0.3)))
        else:
            s = rand_seq(rng, max(min_len, rand_len(rng, hi)), alpha)
        if len(s) >= min_len:
            seqs.append(s)
    return seqs


def unique(seqs):
    seen, out = set(), []
    for s in seqs:
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


class Knobs:
    """Random kernel-choice settings for one case (read per call by the library)."""

    def __init__(self, rng, which):
        self.set = {}
        for k in which:
            if rng.random() < 0.5:
                continue
            self.set[k] = str({
                "DM_LEV_GPAR": lambda: rng.randint(0, 5),
                "DM_LEV_WMAX": lambda: rng.choice((1, 2, 3, 5, 8, 12, 16, 24)),
                "DM_NW_SEQ": lambda: rng.randint(0, 1),
                "DM_NW_CLU": lambda: rng.choice((0, 2, 4, 8)),
                "DM_TREE_BG": lambda: rng.randint(0, 1),
                "DM_TREE_CACHE": lambda: rng.choice((0, 10, 12)),
                "DM_NW_TRACE_GB": lambda: rng.choice((0.001, 0.01, 1)),
                "DM_STREAM_CHUNK_BYTES": lambda: rng.choice((4096, 65536, 1 << 20)),
                "DM_STREAM_PACK": lambda: rng.randint(0, 1),
                "DM_STREAM_HOSTPLAN": lambda: rng.randint(0, 1),
                "DM_STREAM_RAW_FRAC": lambda: rng.choice((0, 0.3, 1)),
            }[k]())

    def __enter__(self):
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(self.set)
        return self

    def __exit__(self, *a):
        for k in self.set:
            os.environ.pop(k, None)


class Campaign:
    def __init__(self, seed):
        import oracle
        import paper_2601_15458_b200 as dm
        self.dm, self.ref = dm, oracle.reference()
        self.ctx = dm.default_context(0)
        self.seed = seed
        self.worlds = {}

    def world_ctx(self, k):
        if k == 1:
            return self.ctx
        if k not in self.worlds:
            from paper_2601_15458_b200.dist import simulate_world
            c = self.dm.Context(0)
            simulate_world(c, k)
            self.worlds[k] = c
        return self.worlds[k]

    # -- distances -------------------------------------------------------------------------
    def _pairs(self, rng, seqs, budget_cells):
        n = len(seqs)
        ia, ib, cells = [], [], 0
        lim = rng.choice((1, 7, 100, 3000, 40000))
        while len(ia) < lim and cells < budget_cells:
            a, b = rng.randrange(n), rng.randrange(n)
            ia.append(a)
            ib.append(b)
            cells += len(seqs[a]) * len(seqs[b])
        return np.array(ia, np.uint32), np.array(ib, np.uint32)

    def case_lev(self, rng):
        alpha = ALPHABETS[rng.choice(list(ALPHABETS))]
        hi = rng.choice((40, 300, 1700, 4200, 9000)) if rng.random() < 0.9 else rng.choice((26000, 40000))
        seqs = rand_set(rng, rng.randint(2, 200 if hi < 5000 else 6), hi, alpha)
        ia, ib = self._pairs(rng, seqs, 3e9)
        with Knobs(rng, ("DM_LEV_GPAR", "DM_LEV_WMAX")) as kn:
            got = self.dm.lev_pairs(self.dm.SeqSet(seqs, self.ctx), ia, ib)
        want = self.ref.lev_pairs(seqs, ia, ib)
        bad = np.nonzero(got != want)[0]
        return (f"alpha {len(alpha)} hi {hi} n {len(seqs)} pairs {len(ia)} knobs {kn.set}",
                None if not len(bad) else f"{len(bad)} distances differ, first pair {bad[0]}: "
                f"lens {len(seqs[ia[bad[0]]])},{len(seqs[ib[bad[0]]])} got {got[bad[0]]} want {want[bad[0]]}")

    def case_packed(self, rng):
        alpha = ALPHABETS[rng.choice(("dna", "dna", "dna", "dna5", "aa", "ascii"))]
        hi = rng.choice((40, 300, 1700, 4200))
        npairs = rng.choice((1, 5, 300, 4000))
        seqs, cells = [], 0
        for _ in range(npairs):
            a = rand_seq(rng, rand_len(rng, hi), alpha)
            b = mutate(rng, a, alpha, rng.choice((0.02, 0.06, 0.4))) if rng.random() < 0.8 else \
                rand_seq(rng, rand_len(rng, hi), alpha)
            seqs += [a, b]
            cells += len(a) * len(b)
            if cells > 3e9:
                break
        data = "".join(seqs).encode()
        offs = np.concatenate([[0], np.cumsum([len(s) for s in seqs])]).astype(np.uint64)
        with Knobs(rng, ("DM_LEV_WMAX", "DM_STREAM_CHUNK_BYTES", "DM_STREAM_PACK", "DM_STREAM_HOSTPLAN",
                         "DM_STREAM_RAW_FRAC")) as kn:
            got = self.dm.lev_pairs_packed(data, offs, self.ctx)
        idx = np.arange(len(seqs) // 2, dtype=np.uint32)
        want = self.ref.lev_pairs(seqs, 2 * idx, 2 * idx + 1)
        bad = np.nonzero(got != want)[0]
        return (f"alpha {len(alpha)} hi {hi} pairs {len(idx)} knobs {kn.set}",
                None if not len(bad) else f"{len(bad)} distances differ, first pair {bad[0]} got {got[bad[0]]} "
                f"want {want[bad[0]]}")

    def case_scan(self, rng):
        alpha = ALPHABETS[rng.choice(list(ALPHABETS))]
        seqs = rand_set(rng, rng.randint(2, 300), rng.choice((50, 400, 1700)), alpha)
        origin = rng.randrange(len(seqs))
        members = np.array(rng.sample(range(len(seqs)), rng.randint(1, len(seqs))), np.uint32)
        with Knobs(rng, ("DM_LEV_GPAR", "DM_LEV_WMAX")) as kn:
            got = self.dm.lev_one_to_many(self.dm.SeqSet(seqs, self.ctx), origin, members)
        want = self.ref.lev_pairs(seqs, np.full(len(members), origin, np.uint32), members)
        return (f"alpha {len(alpha)} n {len(seqs)} members {len(members)} knobs {kn.set}",
                None if np.array_equal(got, want) else "distances differ")

    # -- pairwise aligner ------------------------------------------------------------------
    def _scheme(self, rng):
        dm = self.dm
        go = -rng.randint(0, 14)
        ge = -rng.randint(0, min(4, -go)) if go else 0
        mode = rng.choice(("affine", "affine", "flat"))
        kind = rng.choice(("nt", "nt", "aa", "custom"))
        if kind == "nt":
            return dm.ScoringScheme.nucleotide(go, ge, mode), dict(kind="nt"), "ACGT" if rng.random() < 0.7 else ALPHABETS["iupac"], go, ge, mode
        if kind == "aa":
            return dm.ScoringScheme.protein(go, ge, mode), dict(kind="aa"), ALPHABETS["aa"] if rng.random() < 0.7 else ALPHABETS["aa24"], go, ge, mode
        k = rng.choice((2, 3, 5, 9, 26, 60))
        syms = "".join(rng.sample(ALPHABETS["ascii"], k))
        big = rng.random() < 0.1
        m = [[0] * k for _ in range(k)]
        for i in range(k):
            for j in range(i, k):
                v = rng.randint(-3000, 3000) if big else rng.randint(-6, 9)
                m[i][j] = m[j][i] = v
        flatm = [v for row in m for v in row]
        return (dm.ScoringScheme.custom(syms, flatm, go, ge, mode), dict(kind="custom", symbols=syms, matrix=flatm),
                syms, go, ge, mode)

    def case_nw(self, rng):
        sc, rkw, alpha, go, ge, mode = self._scheme(rng)
        hi = rng.choice((12, 80, 700, 1400, 2700))
        count = rng.choice((1, 3, 20, 70, 700))
        gappy = rng.random() < 0.4  # child center rows carry '-' (msa_merge.cpp:80-83)
        pairs, cells = [], 0
        while len(pairs) < count and cells < 6e7:
            a = rand_seq(rng, max(1, rand_len(rng, hi)), alpha)
            b = mutate(rng, a, alpha, rng.choice((0.03, 0.1, 0.5))) if rng.random() < 0.7 else \
                rand_seq(rng, max(1, rand_len(rng, hi)), alpha)
            if gappy:
                a, b = mutate(rng, a, "-", 0.1), mutate(rng, b, "-", 0.1)
            a, b = a or alpha[0], b or alpha[0]
            pairs.append((a, b))
            cells += len(a) * len(b)
        with Knobs(rng, ("DM_NW_SEQ", "DM_NW_CLU", "DM_NW_TRACE_GB")) as kn:
            got = self.dm.nw_batch(pairs, sc, self.ctx)
        desc = f"{rkw['kind']} K {len(alpha)} go {go} ge {ge} {mode} hi {hi} pairs {len(pairs)} gappy {gappy} knobs {kn.set}"
        for k, ((a, b), g) in enumerate(zip(pairs, got)):
            w = self.ref.nw_align(a, b, gap_open=go, gap_extend=ge, flat=mode == "flat", **rkw)
            if (g.score, g.aligned_a, g.aligned_b, list(g.gaps_into_a), list(g.gaps_into_b)) != \
                    (w["score"], w["aligned_a"], w["aligned_b"], w["gaps_into_a"], w["gaps_into_b"]):
                return desc, f"pair {k} ({len(a)} x {len(b)}): score {g.score} vs {w['score']}"
        return desc, None

    # -- tree / MSA ------------------------------------------------------------------------
    def _family_set(self, rng, alpha, nmax, lmax):
        nfam = rng.randint(1, 6)
        seqs = []
        for _ in range(nfam):
            anc = rand_seq(rng, rng.randint(4, lmax), alpha)
            for _ in range(rng.randint(1, max(1, nmax // nfam))):
                seqs.append(mutate(rng, anc, alpha, rng.choice((0.02, 0.1, 0.3))) or anc)
        seqs = unique([s for s in seqs if s])
        rng.shuffle(seqs)
        return seqs if len(seqs) >= 2 else unique(seqs + [alpha[0], alpha[1]])

    def case_tree(self, rng):
        alpha = ALPHABETS[rng.choice(("dna", "dna", "aa", "iupac", "ascii"))]
        seqs = self._family_set(rng, alpha, rng.choice((6, 40, 300, 1200)), rng.choice((30, 200, 900)))
        seed, cap = rng.choice((42, 0, 7, 2 ** 40 + 3)), rng.choice((2, 5, 16, 100, 128, 200))
        world = rng.choice((1, 1, 2, 3, 8))
        with Knobs(rng, ("DM_TREE_BG", "DM_TREE_CACHE", "DM_LEV_WMAX")) as kn:
            nodes, order = self.dm.build_tree(self.dm.SeqSet(seqs, self.world_ctx(world)), seed=seed, exact_cap=cap)
        rn, ro = self.ref.build_tree(seqs, seed=seed, cap=cap)
        ok = np.array_equal(nodes, rn) and np.array_equal(order, ro)
        return f"alpha {len(alpha)} n {len(seqs)} seed {seed} cap {cap} world {world} knobs {kn.set}", \
            None if ok else "tree differs"

    def case_msa(self, rng):
        kind = rng.choice(("nt", "nt", "aa"))
        alpha = ALPHABETS["dna" if kind == "nt" else "aa"]
        seqs = self._family_set(rng, alpha, rng.choice((5, 30, 150, 500)), rng.choice((20, 150, 700)))
        go = -rng.randint(1, 12)
        ge = -rng.randint(0, min(3, -go))
        mode = rng.choice(("affine", "flat"))
        seed = rng.choice((42, 1, 99))
        world = rng.choice((1, 1, 2, 3, 8))
        sc = (self.dm.ScoringScheme.nucleotide if kind == "nt" else self.dm.ScoringScheme.protein)(go, ge, mode)
        with Knobs(rng, ("DM_TREE_BG", "DM_TREE_CACHE", "DM_NW_SEQ", "DM_NW_CLU", "DM_NW_TRACE_GB")) as kn:
            m = self.dm.msa(self.dm.SeqSet(seqs, self.world_ctx(world)), sc, seed=seed)
        r = self.ref.msa(seqs, kind=kind, gap_open=go, gap_extend=ge, flat=mode == "flat", seed=seed)
        ok = m.width == r["width"] and np.array_equal(m.row_to_sequence, r["row_seq"]) and list(m.rows) == r["rows"]
        return f"{kind} n {len(seqs)} go {go} ge {ge} {mode} seed {seed} world {world} knobs {kn.set}", \
            None if ok else "MSA differs"

    def case_align(self, rng):
        kind = rng.choice(("nt", "aa"))
        alpha = ALPHABETS["dna" if kind == "nt" else "aa"]
        seqs = self._family_set(rng, alpha, rng.choice((5, 40, 200)), rng.choice((20, 200)))
        seqs += [rng.choice(seqs) for _ in range(rng.randint(0, len(seqs)))]  # duplicates re-expanded
        rng.shuffle(seqs)
        if kind == "nt" and rng.random() < 0.15:
            seqs = [s.lower() if rng.random() < 0.5 else s for s in seqs]  # rejected: same error text
        abet = rng.choice(("auto", kind))

        def outcome(f):
            try:
                return ("rows", f())
            except Exception as e:
                return ("error", str(e))

        with Knobs(rng, ("DM_TREE_BG", "DM_NW_SEQ", "DM_NW_CLU")) as kn:
            got = outcome(lambda: self.dm.align(seqs, alphabet=abet, ctx=self.ctx))
        want = outcome(lambda: self.ref.align(seqs, alphabet=abet))
        return f"{kind} n {len(seqs)} alphabet {abet} knobs {kn.set}", \
            None if got == want else f"{got[0]} vs {want[0]}: {str(got[1])[:80]} / {str(want[1])[:80]}"

    # -- FASTA pipeline and metrics (the path's callers) ------------------------
    def case_fasta(self, rng):
        import tempfile
        kind = rng.choice(("nt", "aa"))
        alpha = ALPHABETS["dna" if kind == "nt" else "aa"]
        seqs = self._family_set(rng, alpha, rng.choice((4, 30, 120)), rng.choice((20, 150, 400)))
        seqs += [rng.choice(seqs) for _ in range(rng.randint(0, len(seqs) // 2))]  # duplicates: re-expanded
        rng.shuffle(seqs)
        lines = []
        for k, sq in enumerate(seqs):
            desc = rng.choice(("", " sample", " a  b\tc", " len=%d" % len(sq)))
            lines.append(f">s{k}{desc}")
            if rng.random() < 0.3:
                sq = "".join(c.lower() if rng.random() < 0.5 else c for c in sq)  # normalised by the parser
            w = rng.choice((1, 7, 60, 80, 10 ** 6))
            for x in range(0, len(sq), w):
                lines.append(sq[x:x + w] + rng.choice(("", "", " ", "\r")))
            if rng.random() < 0.2:
                lines.append("")
        text = "\n".join(lines) + rng.choice(("\n", "", "\n\n"))
        abet, order = rng.choice(("auto", kind)), rng.choice(("tree", "input"))
        go = -rng.randint(1, 12)
        ge = -rng.randint(0, min(3, -go))
        mode = rng.choice(("affine", "flat"))
        with tempfile.TemporaryDirectory() as d, Knobs(rng, ("DM_TREE_BG", "DM_NW_SEQ", "DM_NW_CLU")) as kn:
            inp = os.path.join(d, "in.fa")
            with open(inp, "w", newline="") as f:
                f.write(text)

            def side(tag, fn):
                paths = [os.path.join(d, f"{tag}.{x}") for x in ("fa", "tree", "dedup")]
                try:
                    fn(*paths)
                except Exception as e:
                    return ("error", str(e))
                return ("files", [open(q, "rb").read() if os.path.exists(q) else None for q in paths])

            got = side("g", lambda o, t, u: self.dm.run_align(inp, o, alphabet=abet, gap_open=go, gap_extend=ge,
                                                              gap_mode=mode, order=order, dump_tree=t, dump_dedup=u,
                                                              ctx=self.ctx))
            want = side("r", lambda o, t, u: self.ref.run_align(inp, o, alphabet=abet, gap_open=go, gap_extend=ge,
                                                                flat=mode == "flat", order=order, dump_tree=t,
                                                                dump_dedup=u))
        desc = f"{kind} records {len(seqs)} alphabet {abet} order {order} go {go} ge {ge} {mode} knobs {kn.set}"
        if got == want:
            return desc, None
        if got[0] != want[0]:
            return desc, f"{got[0]} vs {want[0]}: {str(got[1])[:80]} / {str(want[1])[:80]}"
        if got[0] == "error":
            return desc, f"error text differs: {got[1][:80]} / {want[1][:80]}"
        which = [n for n, x, y in zip(("fasta", "tree dump", "dedup dump"), got[1], want[1]) if x != y]
        return desc, "differs: " + ", ".join(which)

    def case_metrics(self, rng):
        kind = rng.choice(("nt", "aa"))
        alpha = ALPHABETS["dna" if kind == "nt" else "aa"]
        seqs = self._family_set(rng, alpha, rng.choice((4, 40, 200)), rng.choice((20, 150, 500)))
        sc = (self.dm.ScoringScheme.nucleotide if kind == "nt" else self.dm.ScoringScheme.protein)()
        m = self.dm.msa(self.dm.SeqSet(seqs, self.ctx), sc)
        ss, pb, seed = rng.choice((3, 50, 10000)), rng.choice((1, 20, 100000)), rng.choice((42, 5))
        got = self.dm.evaluate(m, seqs, sample_size=ss, pair_budget=pb, seed=seed, ctx=self.ctx)
        want = self.ref.evaluate(list(m.rows), m.row_to_sequence, seqs, sample_size=ss, pair_budget=pb, seed=seed)
        fields = ("width", "stretch", "gap_percent", "distortion", "p_min", "p_avg", "p_max", "sample_size",
                  "pair_count", "seed", "zero_distance_pairs")
        bad = [k for k in fields if got[k] != want[k]]
        return f"{kind} n {len(seqs)} sample {ss} budget {pb} seed {seed}", \
            None if not bad else f"fields differ: {[(k, got[k], want[k]) for k in bad][:3]}"


    CASES = ("lev", "packed", "scan", "nw", "tree", "msa", "align", "fasta", "metrics")

    def run(self, seconds, kinds=None, log=print, max_cases=None):
        kinds = list(kinds or self.CASES)
        t_end = time.time() + seconds
        counts = {k: 0 for k in kinds}
        failures = []
        case = 0
        while time.time() < t_end and (max_cases is None or case < max_cases):
            kind = kinds[case % len(kinds)]
            rng = random.Random(f"{self.seed}/{case}")
            try:
                desc, err = getattr(self, "case_" + kind)(rng)
            except Exception as e:  # a library error on a valid input is a failure too
                desc, err = "(raised)", f"{type(e).__name__}: {e}"
            counts[kind] += 1
            if err:
                failures.append((case, kind, desc, err))
                log(f"FAIL seed {self.seed} case {case} [{kind}] {desc}: {err}")
            case += 1
        return counts, failures


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=60)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--kinds", default="")
    ap.add_argument("--case", type=int, default=None, help="re-run one case number")
    a = ap.parse_args()
    c = Campaign(a.seed)
    kinds = [k for k in a.kinds.split(",") if k] or None
    if a.case is not None:
        ks = list(kinds or c.CASES)
        kind = ks[a.case % len(ks)]
        print(kind, *getattr(c, "case_" + kind)(random.Random(f"{a.seed}/{a.case}")))
        return 0
    counts, failures = c.run(a.seconds, kinds)
    print(f"fuzz seed {a.seed}: cases {counts}, {len(failures)} failure(s)")
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
