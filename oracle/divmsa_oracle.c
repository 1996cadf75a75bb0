/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 * Plain-C restatement of the reference hot path; see divmsa_oracle.h.
 * Citations are /root/reference/proj file:line. Pure, single-threaded and
 * deliberately direct: it is the yardstick, so it takes no shortcuts. */
#include "divmsa_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

uint64_t orc_mix_seed(uint64_t x) { /* rng.hpp:14-19 (splitmix64 finalizer) */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t orc_combine_seed(uint64_t seed, uint64_t salt) { /* rng.hpp:21-23 */
    return orc_mix_seed(seed ^ orc_mix_seed(salt));
}

/* std::mt19937_64: w=64 n=312 m=156 r=31, a=0xB5026F5AA96619E9,
 * u=29 d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000 t=37
 * c=0xFFF7EEE000000000 l=43 f=6364136223846793005. */
void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

uint64_t orc_bounded_draw(orc_mt64* g, uint64_t bound) { /* rng.hpp:27-35 */
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t v;
    do {
        v = orc_mt64_next(g);
    } while (v >= limit);
    return v % bound;
}

static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? -1 : a > b;
}

uint64_t orc_sample_distinct(orc_mt64* g, uint64_t n, uint64_t k, uint64_t* out) {
    /* rng.hpp:39-59: Floyd's algorithm; the set is emitted sorted. */
    if (k >= n) {
        for (uint64_t i = 0; i < n; ++i) out[i] = i;
        return n;
    }
    uint64_t cnt = 0;
    for (uint64_t j = n - k; j < n; ++j) {
        const uint64_t t = orc_bounded_draw(g, j + 1);
        int seen = 0;
        for (uint64_t q = 0; q < cnt; ++q)
            if (out[q] == t) { seen = 1; break; }
        out[cnt++] = seen ? j : t;
    }
    qsort(out, cnt, sizeof(uint64_t), cmp_u64);
    return cnt;
}

/* ---------------------------------------------------------- distance.cpp */

uint32_t orc_levenshtein(const char* a, size_t na, const char* b, size_t nb) {
    /* distance.cpp:9-48: shorter string as the DP row, exact prefix/suffix
     * trim, two-row unit-cost DP. */
    if (na < nb) {
        const char* t = a; a = b; b = t;
        size_t tn = na; na = nb; nb = tn;
    }
    size_t pre = 0;
    while (pre < nb && a[pre] == b[pre]) ++pre;
    a += pre; b += pre; na -= pre; nb -= pre;
    size_t suf = 0;
    while (suf < nb && a[na - 1 - suf] == b[nb - 1 - suf]) ++suf;
    na -= suf; nb -= suf;
    if (nb == 0) return (uint32_t)na;
    uint32_t* row = (uint32_t*)malloc((nb + 1) * sizeof(uint32_t));
    for (size_t j = 0; j <= nb; ++j) row[j] = (uint32_t)j;
    for (size_t i = 0; i < na; ++i) {
        uint32_t diag = row[0];
        row[0] = (uint32_t)(i + 1);
        uint32_t left = row[0];
        const char ai = a[i];
        for (size_t j = 0; j < nb; ++j) {
            const uint32_t up = row[j + 1];
            const uint32_t sub = diag + (ai != b[j]);
            const uint32_t ul = (up < left ? up : left) + 1;
            const uint32_t best = sub < ul ? sub : ul;
            row[j + 1] = best;
            left = best;
            diag = up;
        }
    }
    const uint32_t d = row[nb];
    free(row);
    return d;
}

/* ------------------------------------------------------ cluster_tree.cpp */

uint64_t orc_hash_members(const uint32_t* members, size_t n) { /* :18-27 FNV-1a */
    uint64_t h = 14695981039346656037ULL;
    for (size_t i = 0; i < n; ++i) {
        h ^= members[i];
        h *= 1099511628211ULL;
    }
    return h;
}

static uint32_t lev_idx(const char* const* seqs, const uint32_t* lens, uint32_t x, uint32_t y) {
    return orc_levenshtein(seqs[x], lens[x], seqs[y], lens[y]);
}

int orc_geometric_median(const uint32_t* members, size_t n, const char* const* seqs,
                         const uint32_t* lens, uint64_t seed, size_t exact_cap,
                         uint32_t* out) {
    /* cluster_tree.cpp:115-166 */
    if (n == 0) return -1;
    if (n == 1) { *out = members[0]; return 0; }
    if (exact_cap < 2) exact_cap = 2;
    uint32_t* cand;
    size_t k;
    if (n <= exact_cap) {
        k = n;
        cand = (uint32_t*)malloc(k * sizeof(uint32_t));
        memcpy(cand, members, k * sizeof(uint32_t));
    } else {
        orc_mt64 g;
        orc_mt64_seed(&g, seed);
        uint64_t* pos = (uint64_t*)malloc(exact_cap * sizeof(uint64_t));
        k = (size_t)orc_sample_distinct(&g, n, exact_cap, pos);
        cand = (uint32_t*)malloc(k * sizeof(uint32_t));
        for (size_t i = 0; i < k; ++i) cand[i] = members[pos[i]];
        free(pos);
    }
    uint32_t* dist = (uint32_t*)calloc(k * k, sizeof(uint32_t));
    for (size_t i = 0; i < k; ++i)
        for (size_t j = i + 1; j < k; ++j) {
            const uint32_t d = lev_idx(seqs, lens, cand[i], cand[j]);
            dist[i * k + j] = d;
            dist[j * k + i] = d;
        }
    size_t best = 0;
    uint64_t best_sum = UINT64_MAX;
    for (size_t i = 0; i < k; ++i) {
        uint64_t sum = 0;
        for (size_t j = 0; j < k; ++j) sum += dist[i * k + j];
        if (sum < best_sum || (sum == best_sum && cand[i] < cand[best])) {
            best_sum = sum;
            best = i;
        }
    }
    *out = cand[best];
    free(dist);
    free(cand);
    return 0;
}

/* :44-54 argmax, ties to the lowest sequence index */
static size_t farthest(const uint32_t* d, const uint32_t* members, size_t n) {
    size_t best = 0;
    for (size_t i = 1; i < n; ++i)
        if (d[i] > d[best] || (d[i] == d[best] && members[i] < members[best])) best = i;
    return best;
}

int orc_build_tree(const char* const* seqs, const uint32_t* lens, size_t n,
                   uint64_t seed, size_t exact_cap, orc_node* nodes, size_t* nnodes,
                   uint32_t* order) {
    /* cluster_tree.cpp:168-235: level-synchronous frontier; children are
     * appended left then right in frontier order. */
    if (n == 0) return 1;
    for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    memset(&nodes[0], 0, sizeof(orc_node));
    nodes[0].begin = 0;
    nodes[0].end = (uint32_t)n;
    nodes[0].center = nodes[0].pole_l = nodes[0].pole_r = 0xffffffffu;
    nodes[0].left = nodes[0].right = nodes[0].parent = -1;
    size_t count = 1;
    size_t fbeg = 0, fend = 1; /* frontier = nodes[fbeg, fend) (BFS numbering) */
    uint32_t* dc = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* dl = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* dr = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* tmp = (uint32_t*)malloc(n * sizeof(uint32_t));
    int rc = 0;
    while (fbeg < fend) {
        const size_t next_begin = count;
        for (size_t f = fbeg; f < fend; ++f) {
            orc_node* nd = &nodes[f];
            const uint32_t* mem = order + nd->begin;
            const size_t m = nd->end - nd->begin;
            if (m == 1) { /* :70-74 leaf */
                nd->center = mem[0];
                continue;
            }
            /* compute_split :76-110 */
            const uint64_t node_seed = orc_combine_seed(seed, orc_hash_members(mem, m));
            uint32_t center;
            orc_geometric_median(mem, m, seqs, lens, node_seed, exact_cap, &center);
            for (size_t i = 0; i < m; ++i) dc[i] = lev_idx(seqs, lens, center, mem[i]);
            uint32_t radius = 0;
            for (size_t i = 0; i < m; ++i) if (dc[i] > radius) radius = dc[i];
            const uint32_t pl = mem[farthest(dc, mem, m)];
            for (size_t i = 0; i < m; ++i) dl[i] = lev_idx(seqs, lens, pl, mem[i]);
            const uint32_t pr = mem[farthest(dl, mem, m)];
            if (pr == pl) { rc = 2; goto done; }
            for (size_t i = 0; i < m; ++i) dr[i] = lev_idx(seqs, lens, pr, mem[i]);
            size_t w = 0;
            for (size_t i = 0; i < m; ++i) if (dl[i] <= dr[i]) tmp[w++] = mem[i];
            const size_t mid = w;
            for (size_t i = 0; i < m; ++i) if (dl[i] > dr[i]) tmp[w++] = mem[i];
            nd->center = center;
            nd->radius = radius;
            nd->pole_l = pl;
            nd->pole_r = pr;
            memcpy(order + nd->begin, tmp, m * sizeof(uint32_t));
            /* :212-231 children, left then right */
            orc_node l, r;
            memset(&l, 0, sizeof l);
            memset(&r, 0, sizeof r);
            l.center = l.pole_l = l.pole_r = r.center = r.pole_l = r.pole_r = 0xffffffffu;
            l.left = l.right = r.left = r.right = -1;
            l.begin = nd->begin;
            l.end = nd->begin + (uint32_t)mid;
            r.begin = l.end;
            r.end = nd->end;
            l.parent = r.parent = (int32_t)f;
            l.depth = r.depth = nd->depth + 1;
            nd->left = (int32_t)count;
            nd->right = (int32_t)count + 1;
            nodes[count++] = l;
            nodes[count++] = r;
        }
        fbeg = next_begin;
        fend = count;
    }
done:
    *nnodes = count;
    free(dc); free(dl); free(dr); free(tmp);
    return rc;
}

/* ---------------------------------------------------------- pairwise.cpp */

static const char kIupacSym[16] = {'A','C','G','T','U','R','Y','S','W','K','M','B','D','H','V','N'};
static const unsigned kIupacMask[16] = {1,2,4,8,8,5,10,6,9,12,3,14,13,11,7,15};

static void table_set(int16_t* t, char x, char y, int v) {
    t[(unsigned char)x * 128 + (unsigned char)y] = (int16_t)v;
    t[(unsigned char)y * 128 + (unsigned char)x] = (int16_t)v;
}

void orc_nucleotide_table(int gap_extend, int16_t* table) {
    /* pairwise.cpp:20-25, :122-137 (+1 if IUPAC sets intersect, else -1) and
     * the gap row of :100-107. */
    memset(table, 0, 128 * 128 * sizeof(int16_t));
    for (int i = 0; i < 16; ++i)
        for (int j = 0; j < 16; ++j)
            table_set(table, kIupacSym[i], kIupacSym[j], (kIupacMask[i] & kIupacMask[j]) ? 1 : -1);
    table_set(table, '-', '-', 0);
    for (int i = 0; i < 16; ++i) table_set(table, '-', kIupacSym[i], gap_extend);
}

/* BLOSUM62 (the standard published matrix) over ARNDCQEGHILKMFPSTWYVBZX*. */
static const char kBloSym[] = "ARNDCQEGHILKMFPSTWYVBZX*";
static const signed char kBlo[24][24] = {
{ 4,-1,-2,-2, 0,-1,-1, 0,-2,-1,-1,-1,-1,-2,-1, 1, 0,-3,-2, 0,-2,-1, 0,-4},
{-1, 5, 0,-2,-3, 1, 0,-2, 0,-3,-2, 2,-1,-3,-2,-1,-1,-3,-2,-3,-1, 0,-1,-4},
{-2, 0, 6, 1,-3, 0, 0, 0, 1,-3,-3, 0,-2,-3,-2, 1, 0,-4,-2,-3, 3, 0,-1,-4},
{-2,-2, 1, 6,-3, 0, 2,-1,-1,-3,-4,-1,-3,-3,-1, 0,-1,-4,-3,-3, 4, 1,-1,-4},
{ 0,-3,-3,-3, 9,-3,-4,-3,-3,-1,-1,-3,-1,-2,-3,-1,-1,-2,-2,-1,-3,-3,-2,-4},
{-1, 1, 0, 0,-3, 5, 2,-2, 0,-3,-2, 1, 0,-3,-1, 0,-1,-2,-1,-2, 0, 3,-1,-4},
{-1, 0, 0, 2,-4, 2, 5,-2, 0,-3,-3, 1,-2,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},
{ 0,-2, 0,-1,-3,-2,-2, 6,-2,-4,-4,-2,-3,-3,-2, 0,-2,-2,-3,-3,-1,-2,-1,-4},
{-2, 0, 1,-1,-3, 0, 0,-2, 8,-3,-3,-1,-2,-1,-2,-1,-2,-2, 2,-3, 0, 0,-1,-4},
{-1,-3,-3,-3,-1,-3,-3,-4,-3, 4, 2,-3, 1, 0,-3,-2,-1,-3,-1, 3,-3,-3,-1,-4},
{-1,-2,-3,-4,-1,-2,-3,-4,-3, 2, 4,-2, 2, 0,-3,-2,-1,-2,-1, 1,-4,-3,-1,-4},
{-1, 2, 0,-1,-3, 1, 1,-2,-1,-3,-2, 5,-1,-3,-1, 0,-1,-3,-2,-2, 0, 1,-1,-4},
{-1,-1,-2,-3,-1, 0,-2,-3,-2, 1, 2,-1, 5, 0,-2,-1,-1,-1,-1, 1,-3,-1,-1,-4},
{-2,-3,-3,-3,-2,-3,-3,-3,-1, 0, 0,-3, 0, 6,-4,-2,-2, 1, 3,-1,-3,-3,-1,-4},
{-1,-2,-2,-1,-3,-1,-1,-2,-2,-3,-3,-1,-2,-4, 7,-1,-1,-4,-3,-2,-2,-1,-2,-4},
{ 1,-1, 1, 0,-1, 0, 0, 0,-1,-2,-2, 0,-1,-2,-1, 4, 1,-3,-2,-2, 0, 0, 0,-4},
{ 0,-1, 0,-1,-1,-1,-1,-2,-2,-1,-1,-1,-1,-2,-1, 1, 5,-2,-2, 0,-1,-1, 0,-4},
{-3,-3,-4,-4,-2,-2,-3,-2,-2,-3,-2,-3,-1, 1,-4,-3,-2,11, 2,-3,-4,-3,-2,-4},
{-2,-2,-2,-3,-2,-1,-2,-3, 2,-1,-1,-2,-1, 3,-3,-2,-2, 2, 7,-1,-3,-2,-1,-4},
{ 0,-3,-3,-3,-1,-2,-2,-3,-3, 3, 1,-2, 1,-1,-2,-2, 0,-3,-1, 4,-3,-2,-1,-4},
{-2,-1, 3, 4,-3, 0, 1,-1, 0,-3,-4, 0,-3,-3,-2, 0,-1,-4,-3,-3, 4, 1,-1,-4},
{-1, 0, 0, 1,-3, 3, 4,-2, 0,-3,-3, 1,-1,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},
{ 0,-1,-1,-1,-2,-1,-1,-1,-1,-1,-1,-1,-1,-1,-2, 0, 0,-2,-1,-1,-1,-1,-1,-4},
{-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4, 1},
};

void orc_protein_table(int gap_extend, int16_t* table) {
    /* pairwise.cpp:27-55, :139-142 and the gap row of :100-107 */
    memset(table, 0, 128 * 128 * sizeof(int16_t));
    for (int i = 0; i < 24; ++i)
        for (int j = 0; j < 24; ++j) table_set(table, kBloSym[i], kBloSym[j], kBlo[i][j]);
    table_set(table, '-', '-', 0);
    for (int i = 0; i < 24; ++i) table_set(table, '-', kBloSym[i], gap_extend);
}

#define ORC_NEG_INF (INT64_MIN / 4) /* pairwise.cpp:266 */

/* pairwise.cpp:272-286: tie order M (0) > GapB (1) > GapA (2) */
static int pick_best(int64_t m, int64_t gb, int64_t ga, int64_t* out) {
    int s = 0;
    *out = m;
    if (gb > *out) { *out = gb; s = 1; }
    if (ga > *out) { *out = ga; s = 2; }
    return s;
}

static void reverse_chars(char* s, size_t n) {
    for (size_t i = 0, j = n; i + 1 < j; ++i, --j) { char t = s[i]; s[i] = s[j - 1]; s[j - 1] = t; }
}
static void reverse_u32(uint32_t* s, size_t n) {
    for (size_t i = 0, j = n; i + 1 < j; ++i, --j) { uint32_t t = s[i]; s[i] = s[j - 1]; s[j - 1] = t; }
}

int orc_nw_align(const char* a, size_t n, const char* b, size_t m,
                 const int16_t* table, int open_surcharge, int gap_extend,
                 int64_t* score, char* out_a, char* out_b, size_t* out_len,
                 uint32_t* gaps_a, size_t* ngaps_a, uint32_t* gaps_b, size_t* ngaps_b) {
    /* pairwise.cpp:301-415 */
    if (n == 0 || m == 0) return 1;
    const int64_t open = open_surcharge, ext = gap_extend;
    int64_t* rm = (int64_t*)malloc((m + 1) * sizeof(int64_t));
    int64_t* rgb = (int64_t*)malloc((m + 1) * sizeof(int64_t));
    int64_t* rga = (int64_t*)malloc((m + 1) * sizeof(int64_t));
    uint8_t* tr = (uint8_t*)malloc((n + 1) * (m + 1));
#define PACK(pm, pgb, pga) (uint8_t)((pm) | ((pgb) << 2) | ((pga) << 4))
    rm[0] = 0; rgb[0] = ORC_NEG_INF; rga[0] = ORC_NEG_INF;
    tr[0] = 0;
    for (size_t j = 1; j <= m; ++j) { /* :322-330 */
        rm[j] = ORC_NEG_INF;
        rgb[j] = ORC_NEG_INF;
        rga[j] = (j == 1 ? open + ext : rga[j - 1] + ext);
        tr[j] = PACK(0, 0, j == 1 ? 0 : 2);
    }
    for (size_t i = 1; i <= n; ++i) {
        int64_t dm = rm[0], dgb = rgb[0], dga = rga[0];
        rm[0] = ORC_NEG_INF;
        rga[0] = ORC_NEG_INF;
        rgb[0] = open + (int64_t)i * ext; /* :338-339 */
        tr[i * (m + 1)] = PACK(0, i == 1 ? 0 : 1, 0);
        const unsigned char ai = (unsigned char)a[i - 1];
        for (size_t j = 1; j <= m; ++j) {
            const int64_t um = rm[j], ugb = rgb[j], uga = rga[j];
            int64_t bm, bgb, bga;
            const int pm = pick_best(dm, dgb, dga, &bm);
            bm += table[ai * 128 + (unsigned char)b[j - 1]];
            const int pgb = pick_best(um + open, ugb, uga + open, &bgb);
            bgb += ext;
            const int pga = pick_best(rm[j - 1] + open, rgb[j - 1] + open, rga[j - 1], &bga);
            bga += ext;
            dm = um; dgb = ugb; dga = uga;
            rm[j] = bm; rgb[j] = bgb; rga[j] = bga;
            tr[i * (m + 1) + j] = PACK(pm, pgb, pga);
        }
    }
    int64_t fs;
    int state = pick_best(rm[m], rgb[m], rga[m], &fs); /* :374-375 */
    *score = fs;
    size_t len = 0, na = 0, nb = 0, i = n, j = m;
    while (i > 0 || j > 0) { /* :384-409 */
        const uint8_t p = tr[i * (m + 1) + j];
        if (state == 0) {
            out_a[len] = a[i - 1]; out_b[len] = b[j - 1]; ++len;
            state = p & 3; --i; --j;
        } else if (state == 1) {
            out_a[len] = a[i - 1]; out_b[len] = '-'; ++len;
            gaps_b[nb++] = (uint32_t)j;
            state = (p >> 2) & 3; --i;
        } else {
            out_a[len] = '-'; out_b[len] = b[j - 1]; ++len;
            gaps_a[na++] = (uint32_t)i;
            state = (p >> 4) & 3; --j;
        }
    }
    reverse_chars(out_a, len); reverse_chars(out_b, len);
    reverse_u32(gaps_a, na); reverse_u32(gaps_b, nb);
    *out_len = len; *ngaps_a = na; *ngaps_b = nb;
#undef PACK
    free(rm); free(rgb); free(rga); free(tr);
    return 0;
}

/* --------------------------------------------------------- msa_merge.cpp */

int orc_insert_gap_columns(const char* rows, size_t nrows, size_t width,
                           const uint32_t* pos, size_t npos, char* out) {
    /* msa_merge.cpp:31-70 */
    for (size_t i = 0; i < npos; ++i) {
        if (pos[i] > width) return 1;
        if (i > 0 && pos[i] < pos[i - 1]) return 2;
    }
    const size_t nw = width + npos;
    for (size_t r = 0; r < nrows; ++r) {
        const char* row = rows + r * width;
        char* o = out + r * nw;
        size_t p = 0, w = 0;
        for (size_t c = 0; c < width; ++c) {
            while (p < npos && pos[p] == c) { o[w++] = '-'; ++p; }
            o[w++] = row[c];
        }
        for (; p < npos; ++p) o[w++] = '-';
    }
    return 0;
}

typedef struct {
    char* data; /* rows x width */
    size_t rows, width;
    uint32_t* seq; /* row -> sequence index */
} block;

static size_t row_of(const block* b, uint32_t s) { /* msa_merge.cpp:9-18 */
    for (size_t i = 0; i < b->rows; ++i)
        if (b->seq[i] == s) return i;
    return (size_t)-1;
}

int orc_align_all(const orc_node* nodes, size_t nnodes, const uint32_t* order,
                  const char* const* seqs, const uint32_t* lens, size_t n,
                  const int16_t* table, int open_surcharge, int gap_extend,
                  char** rows_out, size_t* width_out) {
    /* msa_merge.cpp:107-158. The merge order is schedule-independent
     * (:119-122); children always carry larger BFS ids than their parent
     * (cluster_tree.cpp:225-230), so a reverse sweep over node ids is a valid
     * post-order. */
    (void)order;
    block* blk = (block*)calloc(nnodes, sizeof(block));
    for (size_t v = nnodes; v-- > 0;) {
        const orc_node* nd = &nodes[v];
        if (nd->left < 0) { /* align_leaf :20-29 */
            const uint32_t s = nd->center;
            blk[v].rows = 1;
            blk[v].width = lens[s];
            blk[v].data = (char*)malloc(lens[s] + 1);
            memcpy(blk[v].data, seqs[s], lens[s]);
            blk[v].seq = (uint32_t*)malloc(sizeof(uint32_t));
            blk[v].seq[0] = s;
            continue;
        }
        /* merge :72-105 */
        block* L = &blk[nd->left];
        block* R = &blk[nd->right];
        const size_t lr = row_of(L, nodes[nd->left].center);
        const size_t rr = row_of(R, nodes[nd->right].center);
        const char* ra = L->data + lr * L->width;
        const char* rb = R->data + rr * R->width;
        const size_t cap = L->width + R->width;
        char* oa = (char*)malloc(cap + 1);
        char* ob = (char*)malloc(cap + 1);
        uint32_t* ga = (uint32_t*)malloc((R->width + 1) * sizeof(uint32_t));
        uint32_t* gb = (uint32_t*)malloc((L->width + 1) * sizeof(uint32_t));
        int64_t sc;
        size_t len, nga, ngb;
        orc_nw_align(ra, L->width, rb, R->width, table, open_surcharge, gap_extend, &sc,
                     oa, ob, &len, ga, &nga, gb, &ngb);
        block P;
        P.rows = L->rows + R->rows;
        P.width = len;
        P.data = (char*)malloc(P.rows * len + 1);
        P.seq = (uint32_t*)malloc(P.rows * sizeof(uint32_t));
        orc_insert_gap_columns(L->data, L->rows, L->width, ga, nga, P.data);
        orc_insert_gap_columns(R->data, R->rows, R->width, gb, ngb, P.data + L->rows * len);
        memcpy(P.seq, L->seq, L->rows * sizeof(uint32_t));
        memcpy(P.seq + L->rows, R->seq, R->rows * sizeof(uint32_t));
        free(oa); free(ob); free(ga); free(gb);
        free(L->data); free(L->seq); free(R->data); free(R->seq);
        L->data = R->data = NULL;
        blk[v] = P;
    }
    *rows_out = blk[0].data;
    *width_out = blk[0].width;
    (void)n;
    free(blk[0].seq);
    free(blk);
    return 0;
}

void orc_free(void* p) { free(p); }
