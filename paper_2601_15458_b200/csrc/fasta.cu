// FASTA in and out around the aligner:
//   * parse_fasta_text — the reference's parser (seq_io.cpp:44-119): ids up
//     to the first blank, description after it, residues uppercased with
//     blanks skipped, '\r' stripped, errors "source:line: what". Host code
//     (hashing/parsing on the GPU only pays off at >= 10^6
//     records);
//   * the aligned-FASTA writer (format_fasta / write_fasta, seq_io.cpp:188-225)
//     assembled on the device: one warp per record copies the header and the
//     aligned row with a '\n' every 80 columns straight out of the MSA row
//     buffer (duplicates re-expanded by pointing several records at one
//     row), then one D2H copy and one host write;
//   * run_align (pipeline.cpp:160-187): parse -> align_sequences -> write to
//     "<output>.partial" -> rename, nothing left behind on failure.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "host_copy.h"
#include "capi_guard.h"
#include "pipeline.h"

namespace dm {
namespace {

constexpr uint32_t kLine = 80;  // kFastaLineWidth (seq_io.cpp:13)

struct Record {
    std::string id, description, residues;
};

[[noreturn]] void parse_error(std::string_view source, uint64_t line, const std::string& what) {
    std::ostringstream os;
    os << std::string(source) << ":" << line << ": " << what;
    throw runtime_error(os.str());
}

std::string read_file(const std::string& path) {  // seq_io.cpp:22-33
    std::ifstream in(path, std::ios::binary);
    if (!in) throw runtime_error("cannot open " + path + " for reading");
    std::ostringstream os;
    os << in.rdbuf();
    if (in.bad()) throw runtime_error("I/O error while reading " + path);
    return std::move(os).str();
}

constexpr std::string_view kNucleotide = "ACGTURYSWKMBDHVN";
constexpr std::string_view kProtein = "ARNDCQEGHILKMFPSTWYVBZX*";

// alphabet: -1 structural parse only, 0 nucleotide, 1 protein
std::vector<Record> parse_fasta_text(std::string_view text, int alphabet, bool allow_gaps,
                                     std::string_view source) {
    bool member[256] = {};
    if (alphabet >= 0)
        for (char c : (alphabet == 0 ? kNucleotide : kProtein)) member[(unsigned char)c] = true;
    const char* alpha_name = alphabet == 0 ? "nucleotide" : "protein";
    std::vector<Record> out;
    bool in_record = false;
    uint64_t line_no = 0, record_start = 0;
    auto finish = [&] {
        if (in_record && out.back().residues.empty())
            parse_error(source, record_start, "record '" + out.back().id + "' has no sequence data");
    };
    size_t pos = 0;
    while (pos < text.size()) {
        size_t eol = text.find('\n', pos);
        if (eol == std::string_view::npos) eol = text.size();
        std::string_view line = text.substr(pos, eol - pos);
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        pos = eol + 1;
        ++line_no;
        if (line.empty()) continue;
        if (line.front() == '>') {
            finish();
            std::string_view header = line.substr(1);
            const size_t ws = header.find_first_of(" \t");
            Record r;
            r.id = std::string(header.substr(0, ws));
            if (ws != std::string_view::npos) {
                std::string_view rest = header.substr(ws + 1);
                const size_t first = rest.find_first_not_of(" \t");
                if (first != std::string_view::npos) r.description = std::string(rest.substr(first));
            }
            if (r.id.empty()) parse_error(source, line_no, "header has an empty id");
            out.push_back(std::move(r));
            in_record = true;
            record_start = line_no;
            continue;
        }
        if (!in_record) parse_error(source, line_no, "sequence data before the first '>' header");
        Record& r = out.back();
        r.residues.reserve(r.residues.size() + line.size());
        for (char raw : line) {
            if (std::isspace((unsigned char)raw)) continue;
            const char c = (char)std::toupper((unsigned char)raw);
            if (c == '-') {
                if (!allow_gaps)
                    parse_error(source, line_no, "record '" + r.id + "' contains gap symbol '-' in unaligned input");
            } else if (alphabet >= 0 && !member[(unsigned char)c]) {
                parse_error(source, line_no,
                            "record '" + r.id + "' contains character '" + std::string(1, raw) + "' outside the " +
                                alpha_name + " alphabet");
            }
            r.residues.push_back(c);
        }
    }
    finish();
    if (out.empty()) parse_error(source, line_no, "no FASTA records found");
    return out;
}

// One warp per output record: header bytes, then the residues with a '\n'
// after every 80 of them and after the last (partial) line.
struct FmtRec {
    uint64_t src;   // residues: byte offset into `res`
    uint64_t hdr;   // header (">id[ desc]\n"): byte offset into `hdrs`
    uint64_t out;   // record start in the output
    uint32_t len;   // residues
    uint32_t hlen;  // header bytes
};

__global__ void fasta_format_kernel(const uint8_t* __restrict__ res, const uint8_t* __restrict__ hdrs,
                                    const FmtRec* __restrict__ recs, uint64_t n, uint8_t* __restrict__ out) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp; k < n; k += nwarps) {
        const FmtRec r = recs[k];
        uint8_t* o = out + r.out;
        for (uint32_t t = lane; t < r.hlen; t += 32) o[t] = hdrs[r.hdr + t];
        o += r.hlen;
        const uint32_t body = r.len + (r.len + kLine - 1) / kLine;  // residues + one '\n' per line
        const uint8_t* src = res + r.src;
        for (uint32_t t = lane; t < body; t += 32) {
            const uint32_t line = t / (kLine + 1), c = t % (kLine + 1);
            const uint32_t i = line * kLine + c;
            o[t] = (c < kLine && i < r.len) ? src[i] : (uint8_t)'\n';
        }
    }
}

std::string header_of(const std::string& id, const std::string& desc) {
    std::string h;
    h.reserve(id.size() + desc.size() + 3);
    h.push_back('>');
    h += id;
    if (!desc.empty()) {
        h.push_back(' ');
        h += desc;
    }
    h.push_back('\n');
    return h;
}

// Formats records whose residues sit in device memory `d_res` at
// (src[k], len[k]); returns the FASTA text in host memory.
std::string format_on_device(dm_ctx* ctx, const uint8_t* d_res, const std::vector<std::string>& headers,
                             const std::vector<uint64_t>& src, const std::vector<uint32_t>& len) {
    const uint64_t n = headers.size();
    std::vector<FmtRec> recs(n);
    std::string hdrs;
    uint64_t total = 0;
    for (uint64_t k = 0; k < n; ++k) {
        recs[k] = FmtRec{src[k], hdrs.size(), total, len[k], (uint32_t)headers[k].size()};
        hdrs += headers[k];
        total += headers[k].size() + len[k] + (len[k] + kLine - 1) / kLine;
    }
    std::string text(total, '\0');
    if (n == 0) return text;
    uint8_t* d_hdr = (uint8_t*)ctx->aux.get(hdrs.size() + 1);
    FmtRec* d_recs = (FmtRec*)ctx->aux2.get(n * sizeof(FmtRec));
    uint8_t* d_out = (uint8_t*)ctx->nw_trace.get(total + 1);
    DM_CUDA(cudaMemcpyAsync(d_hdr, hdrs.data(), hdrs.size(), cudaMemcpyHostToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(d_recs, recs.data(), n * sizeof(FmtRec), cudaMemcpyHostToDevice, ctx->stream));
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16));
    fasta_format_kernel<<<grid, 256, 0, ctx->stream>>>(d_res, d_hdr, d_recs, n, d_out);
    DM_CUDA(cudaGetLastError());
    ++ctx->launches;
    {
        uint64_t rd = hdrs.size() + n * sizeof(FmtRec);
        for (uint64_t k = 0; k < n; ++k) rd += len[k];
        trace_bytes("fasta_format_kernel", rd, total);
    }
    download_host(ctx, text.data(), d_out, total, ctx->stream);
    DM_CUDA(cudaStreamSynchronize(ctx->stream));
    return text;
}

// write to "<path>.partial", rename into place (pipeline.cpp:176-186, seq_io.cpp:210-222)
void write_atomically(const std::string& path, const std::string& text) {
    const std::string tmp = path + ".partial";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) throw runtime_error("cannot open " + tmp + " for writing");
    const size_t w = text.empty() ? 0 : std::fwrite(text.data(), 1, text.size(), f);
    const bool ok = w == text.size() && std::fflush(f) == 0;
    std::fclose(f);
    if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) {
        std::remove(tmp.c_str());
        throw runtime_error("I/O error while writing " + tmp);
    }
}

// nlohmann::json::dump() of a string (ensure_ascii = false): '"' '\\' and
// the named control escapes, other bytes < 0x20 as \u00xx, the rest verbatim.
void json_string(std::string& o, std::string_view s) {
    static const char* hex = "0123456789abcdef";
    o.push_back('"');
    for (unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    o += "\\u00";
                    o.push_back(hex[c >> 4]);
                    o.push_back(hex[c & 15]);
                } else {
                    o.push_back((char)c);
                }
        }
    }
    o.push_back('"');
}

// dump_tree (cluster_tree.cpp:253-270): one JSON object per node, keys in
// nlohmann's (sorted) order.
std::string tree_ndjson(const dm_node* nodes, uint64_t nn, const std::vector<std::string>& center_ids) {
    std::string o;
    o.reserve(nn * 96);
    for (uint64_t i = 0; i < nn; ++i) {
        const dm_node& nd = nodes[i];
        o += "{\"cardinality\":" + std::to_string(nd.end - nd.begin) + ",\"center\":";
        json_string(o, center_ids[nd.center]);
        o += ",\"depth\":" + std::to_string(nd.depth) + ",\"node\":" + std::to_string(i) + ",\"parent\":" +
             (nd.parent < 0 ? std::string("null") : std::to_string(nd.parent)) +
             ",\"radius\":" + std::to_string(nd.radius) + "}\n";
    }
    return o;
}

void write_plain(const std::string& path, const std::string& text, const std::string& open_msg,
                 const std::string& io_msg) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw runtime_error(open_msg);
    const size_t w = text.empty() ? 0 : std::fwrite(text.data(), 1, text.size(), f);
    const bool ok = w == text.size() && std::fflush(f) == 0;
    std::fclose(f);
    if (!ok) throw runtime_error(io_msg);
}

}  // namespace
}  // namespace dm

extern "C" {

int dm_run_align(dm_ctx* ctx, const char* input_path, const char* output_path, int alphabet, int gap_open,
                 int gap_extend, int flat, const int16_t* custom_table, const uint8_t* custom_has, uint64_t seed,
                 int input_order, const char* dump_tree_path, const char* dump_dedup_path,
                 dm_align_summary* summary, dm_stats* st) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && input_path && output_path, "null argument");
        const std::string in(input_path);
        // pipeline.cpp:162-170: auto parses structurally, a fixed alphabet validates while parsing
        std::vector<dm::Record> recs =
            dm::parse_fasta_text(dm::read_file(in), alphabet == 1 ? 0 : alphabet == 2 ? 1 : -1, false, in);
        std::string data;
        std::vector<uint64_t> off{0};
        std::vector<std::string> ids;
        ids.reserve(recs.size());
        for (const auto& r : recs) {
            data += r.residues;
            off.push_back(data.size());
            ids.push_back(r.id);
        }
        dm::AlignCore res = dm::align_core(ctx, data.data(), off.data(), (uint32_t)recs.size(), &ids, alphabet,
                                           gap_open, gap_extend, flat, custom_table, custom_has, seed, input_order,
                                           st, false);  // the formatter reads the device rows
        if (dump_dedup_path && *dump_dedup_path) {  // write_dedup_tsv (seq_io.cpp:227-249)
            std::string tsv;
            for (size_t r = 0; r < res.reps.size(); ++r)
                for (uint32_t d : res.dups[r]) tsv += recs[res.reps[r]].id + '\t' + recs[d].id + '\n';
            const std::string p(dump_dedup_path);
            dm::write_plain(p, tsv, "cannot open " + p + " for writing", "I/O error while writing " + p);
        }
        if (dump_tree_path && *dump_tree_path) {  // dump_tree (cluster_tree.cpp:253-280), leaf ids = representatives
            std::vector<std::string> rep_ids(res.reps.size());
            for (size_t r = 0; r < res.reps.size(); ++r) rep_ids[r] = recs[res.reps[r]].id;
            const std::string p(dump_tree_path);
            dm::write_plain(p, dm::tree_ndjson(res.msa->nodes.data(), res.msa->nodes.size(), rep_ids),
                            "cannot open tree dump file: " + p, "failed writing tree dump: " + p);
        }
        const uint64_t n = recs.size(), W = res.msa->width;
        std::vector<std::string> headers(n);
        std::vector<uint64_t> src(n);
        std::vector<uint32_t> len(n, (uint32_t)W);
        for (uint64_t k = 0; k < n; ++k) {
            const dm::Record& r = recs[res.slot_input[k]];
            headers[k] = dm::header_of(r.id, r.description);
            src[k] = (uint64_t)res.slot_row[k] * res.msa->dev_pitch;  // rows still in ctx->rows_a
        }
        const std::string text =
            dm::format_on_device(ctx, (const uint8_t*)ctx->rows_a.p, headers, src, len);
        dm::write_atomically(output_path, text);
        if (summary) *summary = res.summary;  // elapsed_s covers align_sequences, as in the reference
    });
}

int dm_format_tree(const dm_node* nodes, uint64_t nnodes, const char* ids, const uint64_t* id_off, uint64_t nids,
                   char** text, uint64_t* len) {
    return dm::guard([&] {
        dm::require(nodes && id_off && text && len, "null argument");
        std::vector<std::string> v(nids);
        for (uint64_t k = 0; k < nids; ++k) v[k] = std::string(ids + id_off[k], id_off[k + 1] - id_off[k]);
        for (uint64_t i = 0; i < nnodes; ++i)
            if (nodes[i].center >= nids) throw dm::invalid_argument("node center outside the id list");
        const std::string t = dm::tree_ndjson(nodes, nnodes, v);
        char* p = static_cast<char*>(std::malloc(t.size() + 1));
        if (!p) throw std::bad_alloc();
        std::memcpy(p, t.data(), t.size());
        p[t.size()] = 0;
        *text = p;
        *len = t.size();
    });
}

int dm_dump_tree(const dm_node* nodes, uint64_t nnodes, const char* ids, const uint64_t* id_off, uint64_t nids,
                 const char* path) {
    return dm::guard([&] {
        dm::require(nodes && id_off && path, "null argument");
        std::vector<std::string> v(nids);
        for (uint64_t k = 0; k < nids; ++k) v[k] = std::string(ids + id_off[k], id_off[k + 1] - id_off[k]);
        for (uint64_t i = 0; i < nnodes; ++i)
            if (nodes[i].center >= nids) throw dm::invalid_argument("node center outside the id list");
        const std::string p(path);
        dm::write_plain(p, dm::tree_ndjson(nodes, nnodes, v), "cannot open tree dump file: " + p,
                        "failed writing tree dump: " + p);
    });
}

int dm_write_fasta(dm_ctx* ctx, const char* path, const char* ids, const uint64_t* id_off, const char* descs,
                   const uint64_t* desc_off, const char* residues, const uint64_t* res_off, uint64_t n) {
    return dm::guard(ctx, [&] {
        dm::require(ctx && path && id_off && desc_off && res_off, "null argument");
        std::vector<std::string> headers(n);
        std::vector<uint64_t> src(n);
        std::vector<uint32_t> len(n);
        const uint64_t base = res_off[0], nbytes = res_off[n] - base;
        for (uint64_t k = 0; k < n; ++k) {
            headers[k] = dm::header_of(std::string(ids + id_off[k], id_off[k + 1] - id_off[k]),
                                       std::string(descs + desc_off[k], desc_off[k + 1] - desc_off[k]));
            src[k] = res_off[k] - base;
            const uint64_t L = res_off[k + 1] - res_off[k];
            if (L > 0xffffffffull) throw dm::invalid_argument("record longer than 2^32-1 residues");
            len[k] = (uint32_t)L;
        }
        uint8_t* d_res = (uint8_t*)ctx->rows_b.get(nbytes + 1);
        if (nbytes) DM_CUDA(cudaMemcpyAsync(d_res, residues + base, nbytes, cudaMemcpyHostToDevice, ctx->stream));
        dm::write_atomically(path, dm::format_on_device(ctx, d_res, headers, src, len));
    });
}

int dm_parse_fasta(const char* path, int alphabet, int allow_gaps, char** ids, uint64_t** id_off, char** descs,
                   uint64_t** desc_off, char** residues, uint64_t** res_off, uint64_t* n) {
    return dm::guard([&] {
        dm::require(path && ids && id_off && descs && desc_off && residues && res_off && n, "null argument");
        const std::string p(path);
        const auto recs = dm::parse_fasta_text(dm::read_file(p), alphabet == 1 ? 0 : alphabet == 2 ? 1 : -1,
                                               allow_gaps != 0, p);
        *n = recs.size();
        using Field = std::string dm::Record::*;
        const Field fields[3] = {&dm::Record::id, &dm::Record::description, &dm::Record::residues};
        char** datas[3] = {ids, descs, residues};
        uint64_t** offs[3] = {id_off, desc_off, res_off};
        for (int f = 0; f < 3; ++f) {
            uint64_t tot = 0;
            for (const auto& r : recs) tot += (r.*fields[f]).size();
            char* d = (char*)std::malloc(tot + 1);
            uint64_t* o = (uint64_t*)std::malloc((recs.size() + 1) * sizeof(uint64_t));
            if (!d || !o) {
                std::free(d);
                std::free(o);
                throw std::bad_alloc();
            }
            uint64_t at = 0;
            for (size_t k = 0; k < recs.size(); ++k) {
                o[k] = at;
                const std::string& v = recs[k].*fields[f];
                std::memcpy(d + at, v.data(), v.size());
                at += v.size();
            }
            o[recs.size()] = at;
            *datas[f] = d;
            *offs[f] = o;
        }
    });
}

}  // extern "C"
