// Schedule text reader + symbolic planning for the B200 engine.
//
// Reads the reference's canonical `.cgmsched` v1 records (produced by
// ScheduleProgram::serialize, /root/reference/proj/src/schedule.cpp:335-411)
// straight into flat host arrays the device planner uploads; the structural
// checks mirror ScheduleProgram::parse (proj/src/schedule.cpp:413-580).
#include "host_schedule.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace emtb200 {

namespace {

/// Whitespace tokenizer over one line [p, end).
struct Line {
    const char* p;
    const char* end;
    int number;

    bool next(const char*& tok, size_t& len) {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
        if (p >= end) return false;
        tok = p;
        while (p < end && *p != ' ' && *p != '\t' && *p != '\r') ++p;
        len = static_cast<size_t>(p - tok);
        return true;
    }
    bool next_int(long& v) {
        const char* t;
        size_t n;
        if (!next(t, n)) return false;
        char* e = nullptr;
        v = std::strtol(t, &e, 10);
        return e == t + n;
    }
    bool next_double(double& v) {
        const char* t;
        size_t n;
        if (!next(t, n)) return false;
        char* e = nullptr;
        v = std::strtod(t, &e);
        return e == t + n;
    }
    /// "key=<int>"
    bool next_kv(const char* key, long& v) {
        const char* t;
        size_t n;
        if (!next(t, n)) return false;
        const size_t k = std::strlen(key);
        if (n <= k + 1 || std::strncmp(t, key, k) != 0 || t[k] != '=') return false;
        char* e = nullptr;
        v = std::strtol(t + k + 1, &e, 10);
        return e == t + n;
    }
    bool is(const char* tok, size_t len, const char* word) const {
        return std::strlen(word) == len && std::strncmp(tok, word, len) == 0;
    }
};

bool malformed(Failure& f, int line, const std::string& msg) {
    f.code = 1;  // MalformedDocument
    f.where = "line " + std::to_string(line);
    f.message = msg;
    return false;
}

}  // namespace

bool parse_schedule(const char* text, Schedule& s, Failure& fail) {
    const char* p = text;
    const char* text_end = text + std::strlen(text);
    int line_no = 0;
    bool header = false, meta = false, group_open = false;
    int current_layer = -1, last_layer = -1;

    while (p < text_end) {
        const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(text_end - p)));
        if (eol == nullptr) eol = text_end;
        Line ln{p, eol, ++line_no};
        p = eol + 1;
        const char* tag;
        size_t tl;
        if (!ln.next(tag, tl)) continue;

        if (!header) {
            const char *v, *prof;
            size_t vl, pl;
            long layers = 0, width = 0;
            if (!ln.is(tag, tl, "CGMSCHED") || !ln.next(v, vl) || !ln.is(v, vl, "v1") || !ln.next(prof, pl))
                return malformed(fail, line_no, "bad schedule header");
            s.profile.assign(prof, pl);
            if (!ln.next_kv("layers", layers) || !ln.next_kv("width", width))
                return malformed(fail, line_no, "expected layers=<i> width=<i>");
            s.layers = static_cast<int>(layers);
            s.width = static_cast<int>(width);
            if (s.layers < 0 || s.width < 1) return malformed(fail, line_no, "bad layer count or width");
            s.layer_begin.assign(static_cast<size_t>(s.layers) + 1, 0);
            header = true;
            continue;
        }
        if (!meta) {
            if (!ln.is(tag, tl, "META")) return malformed(fail, line_no, "expected META");
            const char* t;
            size_t n;
            if (!ln.next(t, n) || n < 4 || std::strncmp(t, "dt=", 3) != 0) return malformed(fail, line_no, "expected dt=");
            s.dt = std::strtod(t + 3, nullptr);
            long steps, nodes, comps, blocks, extent, consts;
            if (!ln.next_kv("steps", steps) || !ln.next_kv("nodes", nodes) || !ln.next_kv("comps", comps) ||
                !ln.next_kv("blocks", blocks) || !ln.next_kv("extent", extent) || !ln.next_kv("consts", consts))
                return malformed(fail, line_no, "bad META fields");
            s.steps = static_cast<int>(steps);
            s.nodes = static_cast<int>(nodes);
            s.comps = static_cast<int>(comps);
            s.blocks = static_cast<int>(blocks);
            s.extent = static_cast<int>(extent);
            s.consts = static_cast<int>(consts);
            s.const_table.assign(static_cast<size_t>(s.consts) * static_cast<size_t>(s.width), 0.0);
            meta = true;
            continue;
        }

        if (ln.is(tag, tl, "CONST")) {
            long idx;
            if (!ln.next_int(idx) || idx < 0 || idx >= s.consts) return malformed(fail, line_no, "bad CONST index");
            for (int lane = 0; lane < s.width; ++lane) {
                double v;
                if (!ln.next_double(v)) return malformed(fail, line_no, "truncated CONST row");
                s.const_table[static_cast<size_t>(idx) * static_cast<size_t>(s.width) + static_cast<size_t>(lane)] = v;
            }
        } else if (ln.is(tag, tl, "CHANNEL")) {
            const char* name;
            size_t nl;
            long slot;
            if (!ln.next(name, nl) || !ln.next_int(slot)) return malformed(fail, line_no, "bad CHANNEL");
            s.channel_names.emplace_back(name, nl);
            s.channel_slot.push_back(static_cast<int>(slot));
        } else if (ln.is(tag, tl, "LATCH")) {
            long a, b;
            if (!ln.next_int(a) || !ln.next_int(b)) return malformed(fail, line_no, "bad LATCH");
            s.latch_live.push_back(static_cast<int>(a));
            s.latch_shadow.push_back(static_cast<int>(b));
        } else if (ln.is(tag, tl, "MATRIX")) {
            long dim, nnz, lnnz, unnz, v, mat, l, u, scr, dirty, fc;
            if (!ln.next_kv("dim", dim) || !ln.next_kv("nnz", nnz) || !ln.next_kv("lnnz", lnnz) ||
                !ln.next_kv("unnz", unnz) || !ln.next_kv("v", v) || !ln.next_kv("mat", mat) ||
                !ln.next_kv("l", l) || !ln.next_kv("u", u) || !ln.next_kv("scratch", scr) ||
                !ln.next_kv("dirty", dirty) || !ln.next_kv("fcount", fc))
                return malformed(fail, line_no, "bad MATRIX header");
            s.dim = static_cast<int>(dim);
            s.l_nnz = static_cast<int>(lnnz);
            s.u_nnz = static_cast<int>(unnz);
            s.v_base = static_cast<int>(v);
            s.matrix = static_cast<int>(mat);
            s.l = static_cast<int>(l);
            s.u = static_cast<int>(u);
            s.scratch = static_cast<int>(scr);
            s.dirty = static_cast<int>(dirty);
            s.fcount = static_cast<int>(fc);
            s.row_ptr.assign(1, 0);
        } else if (ln.is(tag, tl, "ROW")) {
            long row, col;
            if (!ln.next_int(row)) return malformed(fail, line_no, "bad ROW");
            while (ln.next_int(col)) s.col_idx.push_back(static_cast<int>(col));
            s.row_ptr.push_back(static_cast<int>(s.col_idx.size()));
        } else if (ln.is(tag, tl, "MENTRY")) {
            long idx, slot;
            double sign;
            if (!ln.next_int(idx)) return malformed(fail, line_no, "bad MENTRY");
            while (ln.next_int(slot) && ln.next_double(sign)) {
                s.mentry_slot.push_back(static_cast<int>(slot));
                s.mentry_sign.push_back(sign);
            }
            s.mentry_ptr.push_back(static_cast<int>(s.mentry_slot.size()));
        } else if (ln.is(tag, tl, "GATHER")) {
            long node, slot;
            if (!ln.next_int(node)) return malformed(fail, line_no, "bad GATHER");
            while (ln.next_int(slot)) s.gather_slot.push_back(static_cast<int>(slot));
            s.gather_ptr.push_back(static_cast<int>(s.gather_slot.size()));
        } else if (ln.is(tag, tl, "FINAL")) {
            long idx, v;
            if (!ln.next_int(idx)) return malformed(fail, line_no, "bad FINAL");
            for (int k = 0; k < 5; ++k) {
                if (!ln.next_int(v)) return malformed(fail, line_no, "truncated FINAL");
                s.finalize.push_back(static_cast<int>(v));
            }
        } else if (ln.is(tag, tl, "WATCH")) {
            long slot;
            while (ln.next_int(slot)) s.watch.push_back(static_cast<int>(slot));
        } else if (ln.is(tag, tl, "LAYER")) {
            long idx;
            if (!ln.next_int(idx) || idx < 0 || idx >= s.layers) return malformed(fail, line_no, "layer index out of range");
            current_layer = static_cast<int>(idx);
            for (int k = last_layer + 1; k <= current_layer; ++k)
                s.layer_begin[static_cast<size_t>(k)] = static_cast<int>(s.procs.size());
            last_layer = std::max(last_layer, current_layer);
            group_open = false;
        } else if (ln.is(tag, tl, "GROUP")) {
            if (current_layer < 0) return malformed(fail, line_no, "GROUP before LAYER");
            group_open = true;
        } else if (ln.is(tag, tl, "P")) {
            if (!group_open) return malformed(fail, line_no, "P before GROUP");
            long f[12];
            for (long& x : f)
                if (!ln.next_int(x)) return malformed(fail, line_no, "truncated P record");
            Proc pr;
            pr.id = static_cast<int>(f[0]);
            pr.kind = static_cast<int>(f[1]);
            pr.code = static_cast<int>(f[2]);
            pr.lane = static_cast<int>(f[3]);
            pr.out = static_cast<int>(f[4]);
            pr.out_len = static_cast<int>(f[5]);
            pr.out2 = static_cast<int>(f[6]);
            pr.state = static_cast<int>(f[7]);
            pr.state_len = static_cast<int>(f[8]);
            pr.par = static_cast<int>(f[9]);
            pr.par_len = static_cast<int>(f[10]);
            if (pr.kind < 0 || pr.kind >= 13) return malformed(fail, line_no, "process kind out of range");
            pr.in_base = static_cast<int>(s.port_slot.size());
            pr.in_count = static_cast<int>(f[11]);
            for (long j = 0; j < f[11]; ++j) {
                long slot;
                double sign;
                if (!ln.next_int(slot) || !ln.next_double(sign)) return malformed(fail, line_no, "truncated port list");
                s.port_slot.push_back(static_cast<int>(slot));
                s.port_sign.push_back(sign);
            }
            s.procs.push_back(pr);
        } else {
            return malformed(fail, line_no, "unknown record '" + std::string(tag, tl) + "'");
        }
    }
    if (!meta) return malformed(fail, line_no, "empty schedule");
    for (int k = last_layer + 1; k <= s.layers; ++k) s.layer_begin[static_cast<size_t>(k)] = static_cast<int>(s.procs.size());

    if (static_cast<int>(s.row_ptr.size()) != s.dim + 1) {
        fail = {1, "", "matrix row count does not match dimension"};
        return false;
    }
    if (static_cast<int>(s.mentry_ptr.size()) != static_cast<int>(s.col_idx.size()) + 1 ||
        static_cast<int>(s.gather_ptr.size()) != s.nodes + 1 ||
        static_cast<int>(s.finalize.size()) != 5 * s.comps) {
        fail = {1, "", "solver tables are truncated"};
        return false;
    }
    if (static_cast<int>(s.procs.size()) < 2 + 2 * s.comps) {
        fail = {1, "", "process records are truncated"};
        return false;
    }
    return true;
}

void lu_symbolic(Schedule& s) {
    // Row i's pattern = A's row i + {i} + the tails (cols > c) of settled U rows
    // c < i reached so far; scanning c ascending reproduces the reference's
    // growing std::set walk (proj/src/sparse.cpp:54-66) exactly.
    const int n = s.dim;
    s.l_row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    s.u_row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    s.l_col.clear();
    s.u_col.clear();
    std::vector<char> mark(static_cast<size_t>(n), 0);
    for (int i = 0; i < n; ++i) {
        std::fill(mark.begin(), mark.end(), 0);
        for (int k = s.row_ptr[static_cast<size_t>(i)]; k < s.row_ptr[static_cast<size_t>(i) + 1]; ++k)
            mark[static_cast<size_t>(s.col_idx[static_cast<size_t>(k)])] = 1;
        mark[static_cast<size_t>(i)] = 1;
        for (int c = 0; c < i; ++c) {
            if (!mark[static_cast<size_t>(c)]) continue;
            for (int j = s.u_row_ptr[static_cast<size_t>(c)]; j < s.u_row_ptr[static_cast<size_t>(c) + 1]; ++j) {
                const int col = s.u_col[static_cast<size_t>(j)];
                if (col > c) mark[static_cast<size_t>(col)] = 1;
            }
        }
        for (int c = 0; c < n; ++c) {
            if (!mark[static_cast<size_t>(c)]) continue;
            (c < i ? s.l_col : s.u_col).push_back(c);
        }
        s.l_row_ptr[static_cast<size_t>(i) + 1] = static_cast<int>(s.l_col.size());
        s.u_row_ptr[static_cast<size_t>(i) + 1] = static_cast<int>(s.u_col.size());
    }
}

void triangular_levels(const Schedule& s, std::vector<int>& fwd_ptr, std::vector<int>& fwd_rows,
                       std::vector<int>& bwd_ptr, std::vector<int>& bwd_rows) {
    const int n = s.dim;
    std::vector<int> level(static_cast<size_t>(n), 0);
    int depth = 0;
    for (int i = 0; i < n; ++i) {
        int lv = 0;
        for (int k = s.l_row_ptr[static_cast<size_t>(i)]; k < s.l_row_ptr[static_cast<size_t>(i) + 1]; ++k)
            lv = std::max(lv, level[static_cast<size_t>(s.l_col[static_cast<size_t>(k)])] + 1);
        level[static_cast<size_t>(i)] = lv;
        depth = std::max(depth, lv + 1);
    }
    fwd_ptr.assign(static_cast<size_t>(depth) + 1, 0);
    fwd_rows.clear();
    for (int d = 0; d < depth; ++d) {
        for (int i = 0; i < n; ++i)
            if (level[static_cast<size_t>(i)] == d) fwd_rows.push_back(i);
        fwd_ptr[static_cast<size_t>(d) + 1] = static_cast<int>(fwd_rows.size());
    }
    depth = 0;
    for (int i = n - 1; i >= 0; --i) {
        int lv = 0;
        for (int k = s.u_row_ptr[static_cast<size_t>(i)] + 1; k < s.u_row_ptr[static_cast<size_t>(i) + 1]; ++k)
            lv = std::max(lv, level[static_cast<size_t>(s.u_col[static_cast<size_t>(k)])] + 1);
        level[static_cast<size_t>(i)] = lv;
        depth = std::max(depth, lv + 1);
    }
    bwd_ptr.assign(static_cast<size_t>(depth) + 1, 0);
    bwd_rows.clear();
    for (int d = 0; d < depth; ++d) {
        for (int i = n - 1; i >= 0; --i)
            if (level[static_cast<size_t>(i)] == d) bwd_rows.push_back(i);
        bwd_ptr[static_cast<size_t>(d) + 1] = static_cast<int>(bwd_rows.size());
    }
}

}  // namespace emtb200
