/* Plain-C restatement of the reference's EMT schedule executor.
 *
 * TEST INFRASTRUCTURE ONLY (see emt_oracle.h). This is the CPU checker the
 * CUDA engine is compared against; it is pinned bit-for-bit against the
 * reference library itself (oracle/_ref/libemtref.so, built from
 * /root/reference/proj/src by oracle/Makefile) on the golden cases in
 * tests/golden/ — see tests/test_oracle.py.
 *
 * Every step follows the reference's own operation order; the file:line
 * citations below are into /root/reference/proj. Compile with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:12-15).
 */
#define _POSIX_C_SOURCE 200809L
#include "emt_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ErrorCode + 1 (proj/include/emtgrid/common.hpp:11-33) */
enum {
    ST_OK = 0,
    ST_MALFORMED = 1,
    ST_NONFINITE = 7,
    ST_SINGULAR = 8,
    ST_DIMENSION = 10,
    ST_UNKNOWN_KIND = 14,
};

/* KernelId (proj/include/emtgrid/kernels.hpp:36-59) */
enum {
    K_RES = 0, K_IND, K_CAP, K_SRL, K_VSRC, K_ISRC, K_CSRC, K_SW, K_INJ, K_FACT, K_SOLVE,
    K_GAIN, K_SUM, K_INTEG, K_LAG, K_LIM, K_PI, K_CMP, K_CONST, K_DELAY,
    K_BERG, /* extension (not in the reference): Bergeron line end, see case K_BERG */
    K_COUNT
};

typedef struct {
    int id, kind, code, lane;
    int out, out_len, out2, state, state_len, par, par_len;
    int in_base, in_count;
} proc_t;

struct emto_schedule {
    int width, steps, nodes, comps, blocks, extent, consts, layers;
    double dt;
    double* const_table; /* consts * width */
    int nch;
    int* ch_slot;
    int nlatch;
    int* latch_live;
    int* latch_shadow;
    /* solver tables (proj/include/emtgrid/schedule.hpp:22-39) */
    int dim, nnz, l_nnz, u_nnz, v_base, mat, l, u, scratch, dirty, fcount;
    int* row_ptr; /* dim+1 */
    int* col_idx; /* nnz */
    int* ment_ptr; /* nnz+1 */
    int* ment_slot;
    double* ment_sign;
    int* gat_ptr; /* nodes+1 */
    int* gat_slot;
    int* fin; /* comps x 5: i g h va vb */
    int nwatch;
    int* watch;
    /* processes, layer-major (exec.cpp:31-62 decode) */
    int nproc;
    proc_t* procs;
    int* layer_begin; /* layers+1 */
    int nport;
    int* port_slot;
    double* port_sign;
    /* lu_symbolic (sparse.cpp:44-77) */
    int *l_row_ptr, *l_col, *u_row_ptr, *u_col;
};

/* ------------------------------------------------------------------ util */

typedef struct {
    int* v;
    int n, cap;
} ivec;
typedef struct {
    double* v;
    int n, cap;
} dvec;

static void ipush(ivec* a, int x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->v = (int*)realloc(a->v, sizeof(int) * (size_t)a->cap);
    }
    a->v[a->n++] = x;
}
static void dpush(dvec* a, double x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 16;
        a->v = (double*)realloc(a->v, sizeof(double) * (size_t)a->cap);
    }
    a->v[a->n++] = x;
}

static int set_err(char* err, int err_len, int code, const char* fmt, ...) {
    if (err && err_len > 0) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err, (size_t)err_len, fmt, ap);
        va_end(ap);
    }
    return code;
}

/* "key=value" token -> value (schedule.cpp:386-392) */
static int kv_int(const char* tok, const char* key, int* ok) {
    size_t k = strlen(key);
    if (!tok || strncmp(tok, key, k) != 0 || tok[k] != '=') {
        *ok = 0;
        return 0;
    }
    return atoi(tok + k + 1);
}

void emto_free(emto_schedule* s) {
    if (!s) return;
    free(s->const_table); free(s->ch_slot); free(s->latch_live); free(s->latch_shadow);
    free(s->row_ptr); free(s->col_idx); free(s->ment_ptr); free(s->ment_slot); free(s->ment_sign);
    free(s->gat_ptr); free(s->gat_slot); free(s->fin); free(s->watch); free(s->procs);
    free(s->layer_begin); free(s->port_slot); free(s->port_sign);
    free(s->l_row_ptr); free(s->l_col); free(s->u_row_ptr); free(s->u_col);
    free(s);
}

/* lu_symbolic: row-by-row reachability, identity ordering, diagonal first in
 * each U row (proj/src/sparse.cpp:44-77). Scanning columns c < i in
 * ascending order and OR-ing U row c's tail is exactly the std::set walk
 * of the reference (insertions only add columns > c). */
static void lu_symbolic(emto_schedule* s) {
    const int n = s->dim;
    ivec lc = {0}, uc = {0};
    s->l_row_ptr = (int*)calloc((size_t)n + 1, sizeof(int));
    s->u_row_ptr = (int*)calloc((size_t)n + 1, sizeof(int));
    char* mark = (char*)calloc((size_t)n + 1, 1);
    for (int i = 0; i < n; ++i) {
        memset(mark, 0, (size_t)n);
        for (int k = s->row_ptr[i]; k < s->row_ptr[i + 1]; ++k) mark[s->col_idx[k]] = 1;
        mark[i] = 1;
        for (int c = 0; c < i; ++c) {
            if (!mark[c]) continue;
            for (int j = s->u_row_ptr[c]; j < s->u_row_ptr[c + 1]; ++j) {
                if (uc.v[j] > c) mark[uc.v[j]] = 1;
            }
        }
        for (int c = 0; c < n; ++c) {
            if (!mark[c]) continue;
            if (c < i) ipush(&lc, c); else ipush(&uc, c);
        }
        s->l_row_ptr[i + 1] = lc.n;
        s->u_row_ptr[i + 1] = uc.n;
    }
    free(mark);
    s->l_col = lc.v;
    s->u_col = uc.v;
}

/* ScheduleProgram::parse (proj/src/schedule.cpp:413-580); record grammar in
 * proj/docs/schedule_format.md. */
int emto_parse(const char* text, emto_schedule** out, char* err, int err_len) {
    emto_schedule* s = (emto_schedule*)calloc(1, sizeof(emto_schedule));
    char* buf = strdup(text);
    char* save_line = NULL;
    int line_no = 0, ok = 1, rc = ST_OK;
    int have_header = 0, have_meta = 0;
    ivec chs = {0}, lat_l = {0}, lat_s = {0}, rowp = {0}, cols = {0}, mptr = {0}, mslot = {0};
    dvec msign = {0};
    ivec gptr = {0}, gslot = {0}, fin = {0}, watch = {0}, ports = {0}, lbeg = {0};
    dvec psign = {0};
    proc_t* procs = NULL;
    int nproc = 0, cap_proc = 0, cur_layer = -1, group_open = 0, last_layer_seen = -1;

    ipush(&mptr, 0);
    ipush(&gptr, 0);
    for (char* line = strtok_r(buf, "\n", &save_line); line; line = strtok_r(NULL, "\n", &save_line)) {
        ++line_no;
        char* save_tok = NULL;
        char* tag = strtok_r(line, " \t\r", &save_tok);
        if (!tag) continue;
#define NEXT() strtok_r(NULL, " \t\r", &save_tok)
        if (!have_header) {
            char* ver = NEXT();
            char* prof = NEXT();
            if (strcmp(tag, "CGMSCHED") != 0 || !ver || strcmp(ver, "v1") != 0 || !prof) {
                rc = set_err(err, err_len, ST_MALFORMED, "bad schedule header (at line %d)", line_no);
                goto fail;
            }
            s->layers = kv_int(NEXT(), "layers", &ok);
            s->width = kv_int(NEXT(), "width", &ok);
            if (!ok) { rc = set_err(err, err_len, ST_MALFORMED, "bad header fields (at line %d)", line_no); goto fail; }
            have_header = 1;
            continue;
        }
        if (!have_meta) {
            if (strcmp(tag, "META") != 0) { rc = set_err(err, err_len, ST_MALFORMED, "expected META (at line %d)", line_no); goto fail; }
            char* t = NEXT();
            if (!t || strncmp(t, "dt=", 3) != 0) { rc = set_err(err, err_len, ST_MALFORMED, "expected dt="); goto fail; }
            s->dt = strtod(t + 3, NULL);
            s->steps = kv_int(NEXT(), "steps", &ok);
            s->nodes = kv_int(NEXT(), "nodes", &ok);
            s->comps = kv_int(NEXT(), "comps", &ok);
            s->blocks = kv_int(NEXT(), "blocks", &ok);
            s->extent = kv_int(NEXT(), "extent", &ok);
            s->consts = kv_int(NEXT(), "consts", &ok);
            if (!ok) { rc = set_err(err, err_len, ST_MALFORMED, "bad META (at line %d)", line_no); goto fail; }
            s->const_table = (double*)calloc((size_t)s->consts * (size_t)s->width + 1, sizeof(double));
            for (int l = 0; l <= s->layers; ++l) ipush(&lbeg, 0);
            have_meta = 1;
            continue;
        }
        if (!strcmp(tag, "CONST")) {
            int idx = atoi(NEXT());
            for (int lane = 0; lane < s->width; ++lane) {
                char* t = NEXT();
                if (!t) { rc = set_err(err, err_len, ST_MALFORMED, "truncated CONST (at line %d)", line_no); goto fail; }
                s->const_table[(size_t)idx * (size_t)s->width + (size_t)lane] = strtod(t, NULL);
            }
        } else if (!strcmp(tag, "CHANNEL")) {
            (void)NEXT();
            ipush(&chs, atoi(NEXT()));
        } else if (!strcmp(tag, "LATCH")) {
            ipush(&lat_l, atoi(NEXT()));
            ipush(&lat_s, atoi(NEXT()));
        } else if (!strcmp(tag, "MATRIX")) {
            s->dim = kv_int(NEXT(), "dim", &ok);
            (void)NEXT(); /* nnz implied by rows */
            s->l_nnz = kv_int(NEXT(), "lnnz", &ok);
            s->u_nnz = kv_int(NEXT(), "unnz", &ok);
            s->v_base = kv_int(NEXT(), "v", &ok);
            s->mat = kv_int(NEXT(), "mat", &ok);
            s->l = kv_int(NEXT(), "l", &ok);
            s->u = kv_int(NEXT(), "u", &ok);
            s->scratch = kv_int(NEXT(), "scratch", &ok);
            s->dirty = kv_int(NEXT(), "dirty", &ok);
            s->fcount = kv_int(NEXT(), "fcount", &ok);
            if (!ok) { rc = set_err(err, err_len, ST_MALFORMED, "bad MATRIX (at line %d)", line_no); goto fail; }
            rowp.n = 0;
            ipush(&rowp, 0);
        } else if (!strcmp(tag, "ROW")) {
            (void)NEXT();
            for (char* t = NEXT(); t; t = NEXT()) ipush(&cols, atoi(t));
            ipush(&rowp, cols.n);
        } else if (!strcmp(tag, "MENTRY")) {
            (void)NEXT();
            for (char* t = NEXT(); t; t = NEXT()) {
                char* sg = NEXT();
                if (!sg) break;
                ipush(&mslot, atoi(t));
                dpush(&msign, strtod(sg, NULL));
            }
            ipush(&mptr, mslot.n);
        } else if (!strcmp(tag, "GATHER")) {
            (void)NEXT();
            for (char* t = NEXT(); t; t = NEXT()) ipush(&gslot, atoi(t));
            ipush(&gptr, gslot.n);
        } else if (!strcmp(tag, "FINAL")) {
            (void)NEXT();
            for (int k = 0; k < 5; ++k) ipush(&fin, atoi(NEXT()));
        } else if (!strcmp(tag, "WATCH")) {
            for (char* t = NEXT(); t; t = NEXT()) ipush(&watch, atoi(t));
        } else if (!strcmp(tag, "LAYER")) {
            cur_layer = atoi(NEXT());
            group_open = 0;
            if (cur_layer < 0 || cur_layer >= s->layers) {
                rc = set_err(err, err_len, ST_MALFORMED, "layer index out of range (at line %d)", line_no);
                goto fail;
            }
            /* layers are emitted in order; record the flattened start */
            for (int l = last_layer_seen + 1; l <= cur_layer; ++l) lbeg.v[l] = nproc;
            last_layer_seen = cur_layer;
        } else if (!strcmp(tag, "GROUP")) {
            if (cur_layer < 0) { rc = set_err(err, err_len, ST_MALFORMED, "GROUP before LAYER"); goto fail; }
            group_open = 1;
        } else if (!strcmp(tag, "P")) {
            if (!group_open) { rc = set_err(err, err_len, ST_MALFORMED, "P before GROUP"); goto fail; }
            if (nproc == cap_proc) {
                cap_proc = cap_proc ? 2 * cap_proc : 64;
                procs = (proc_t*)realloc(procs, sizeof(proc_t) * (size_t)cap_proc);
            }
            proc_t* p = &procs[nproc++];
            int f[12];
            for (int k = 0; k < 12; ++k) {
                char* t = NEXT();
                if (!t) { rc = set_err(err, err_len, ST_MALFORMED, "truncated P (at line %d)", line_no); goto fail; }
                f[k] = atoi(t);
            }
            p->id = f[0]; p->kind = f[1]; p->code = f[2]; p->lane = f[3];
            p->out = f[4]; p->out_len = f[5]; p->out2 = f[6]; p->state = f[7];
            p->state_len = f[8]; p->par = f[9]; p->par_len = f[10];
            if (p->kind < 0 || p->kind >= 13) { rc = set_err(err, err_len, ST_MALFORMED, "process kind out of range"); goto fail; }
            p->in_base = ports.n;
            p->in_count = f[11];
            for (int j = 0; j < f[11]; ++j) {
                char* a = NEXT();
                char* b = NEXT();
                if (!a || !b) { rc = set_err(err, err_len, ST_MALFORMED, "truncated port list (at line %d)", line_no); goto fail; }
                ipush(&ports, atoi(a));
                dpush(&psign, strtod(b, NULL));
            }
        } else {
            rc = set_err(err, err_len, ST_MALFORMED, "unknown record '%s' (at line %d)", tag, line_no);
            goto fail;
        }
#undef NEXT
    }
    if (!have_meta) { rc = set_err(err, err_len, ST_MALFORMED, "empty schedule"); goto fail; }
    for (int l = last_layer_seen + 1; l <= s->layers; ++l) lbeg.v[l] = nproc;
    s->nch = chs.n; s->ch_slot = chs.v; chs.v = NULL;
    s->nlatch = lat_l.n; s->latch_live = lat_l.v; s->latch_shadow = lat_s.v; lat_l.v = lat_s.v = NULL;
    s->row_ptr = rowp.v; s->col_idx = cols.v; s->nnz = cols.n; rowp.v = cols.v = NULL;
    if (rowp.n != s->dim + 1) { rc = set_err(err, err_len, ST_MALFORMED, "matrix row count does not match dimension"); goto fail; }
    s->ment_ptr = mptr.v; s->ment_slot = mslot.v; s->ment_sign = msign.v; mptr.v = mslot.v = NULL; msign.v = NULL;
    s->gat_ptr = gptr.v; s->gat_slot = gslot.v; gptr.v = gslot.v = NULL;
    s->fin = fin.v; fin.v = NULL;
    s->nwatch = watch.n; s->watch = watch.v; watch.v = NULL;
    s->procs = procs; s->nproc = nproc; procs = NULL;
    s->layer_begin = lbeg.v; lbeg.v = NULL;
    s->nport = ports.n; s->port_slot = ports.v; s->port_sign = psign.v; ports.v = NULL; psign.v = NULL;
    if (mptr.n != s->nnz + 1 || gptr.n != s->nodes + 1 || fin.n != 5 * s->comps) {
        rc = set_err(err, err_len, ST_MALFORMED, "solver tables are truncated");
        goto fail;
    }
    if (s->nproc < 2 + 2 * s->comps) { rc = set_err(err, err_len, ST_MALFORMED, "process records are truncated"); goto fail; }
    lu_symbolic(s);
    free(buf);
    *out = s;
    return ST_OK;
fail:
    free(buf);
    free(chs.v); free(lat_l.v); free(lat_s.v); free(rowp.v); free(cols.v); free(mptr.v); free(mslot.v);
    free(msign.v); free(gptr.v); free(gslot.v); free(fin.v); free(watch.v); free(ports.v); free(psign.v);
    free(lbeg.v); free(procs);
    emto_free(s);
    *out = NULL;
    return rc;
}

void emto_shape(const emto_schedule* s, int* width, int* channels, int* extent, int* steps,
                int* nodes, int* l_nnz, int* u_nnz) {
    if (width) *width = s->width;
    if (channels) *channels = s->nch;
    if (extent) *extent = s->extent;
    if (steps) *steps = s->steps;
    if (nodes) *nodes = s->nodes;
    if (l_nnz) *l_nnz = s->l_row_ptr[s->dim];
    if (u_nnz) *u_nnz = s->u_row_ptr[s->dim];
}

/* ------------------------------------------------------------------ engine */

typedef struct {
    const emto_schedule* s;
    double* arena;
    const double* consts;
    int w;
    int32_t* events;
    int max_events;
    int n_events;
    int err_index, err_lane;
} eng_t;

/* Engine::read: slot -1 is the ground sentinel 0.0 (exec.cpp:73-75) */
static inline double rd(const eng_t* e, int slot, int lane) {
    return slot < 0 ? 0.0 : e->arena[(size_t)slot * (size_t)e->w + (size_t)lane];
}

/* lu_factor (proj/src/sparse.cpp:79-145), lane-batched, up-looking rows,
 * unit L, no pivoting; SingularMatrix when |u_ii| <= 1e-12 max|A_lane|. */
static int lu_factor(eng_t* e, char* err, int err_len) {
    const emto_schedule* s = e->s;
    const int n = s->dim;
    const size_t w = (size_t)e->w;
    const double* a = e->arena + (size_t)s->mat * w;
    double* lv = e->arena + (size_t)s->l * w;
    double* uv = e->arena + (size_t)s->u * w;
    double* scr = e->arena + (size_t)s->scratch * w;
    double* max_abs = (double*)calloc(w, sizeof(double));
    for (int k = 0; k < s->nnz; ++k) {
        for (size_t lane = 0; lane < w; ++lane) {
            const double x = fabs(a[(size_t)k * w + lane]);
            max_abs[lane] = max_abs[lane] < x ? x : max_abs[lane]; /* std::max(a,b): a<b?b:a */
        }
    }
    for (int i = 0; i < n; ++i) {
        for (int k = s->l_row_ptr[i]; k < s->l_row_ptr[i + 1]; ++k)
            for (size_t lane = 0; lane < w; ++lane) scr[(size_t)s->l_col[k] * w + lane] = 0.0;
        for (int k = s->u_row_ptr[i]; k < s->u_row_ptr[i + 1]; ++k)
            for (size_t lane = 0; lane < w; ++lane) scr[(size_t)s->u_col[k] * w + lane] = 0.0;
        for (int k = s->row_ptr[i]; k < s->row_ptr[i + 1]; ++k)
            for (size_t lane = 0; lane < w; ++lane)
                scr[(size_t)s->col_idx[k] * w + lane] = a[(size_t)k * w + lane];
        for (int k = s->l_row_ptr[i]; k < s->l_row_ptr[i + 1]; ++k) {
            const int col = s->l_col[k];
            const int ub = s->u_row_ptr[col];
            const double* ud = uv + (size_t)ub * w;
            double* lik = lv + (size_t)k * w;
            double* wc = scr + (size_t)col * w;
            for (size_t lane = 0; lane < w; ++lane) lik[lane] = wc[lane] / ud[lane];
            for (int j = ub + 1; j < s->u_row_ptr[col + 1]; ++j) {
                double* wj = scr + (size_t)s->u_col[j] * w;
                const double* ukj = uv + (size_t)j * w;
                for (size_t lane = 0; lane < w; ++lane) wj[lane] -= lik[lane] * ukj[lane];
            }
        }
        for (int k = s->u_row_ptr[i]; k < s->u_row_ptr[i + 1]; ++k)
            for (size_t lane = 0; lane < w; ++lane)
                uv[(size_t)k * w + lane] = scr[(size_t)s->u_col[k] * w + lane];
        const double* diag = uv + (size_t)s->u_row_ptr[i] * w;
        for (size_t lane = 0; lane < w; ++lane) {
            if (!(fabs(diag[lane]) > 1e-12 * max_abs[lane])) {
                free(max_abs);
                e->err_index = i;
                e->err_lane = (int)lane;
                return set_err(err, err_len, ST_SINGULAR, "zero pivot below tolerance in lane %d (at row %d)",
                               (int)lane, i);
            }
        }
    }
    free(max_abs);
    return ST_OK;
}

/* lu_solve (proj/src/sparse.cpp:147-172): forward (unit L), backward (U). */
static void lu_solve(eng_t* e) {
    const emto_schedule* s = e->s;
    const size_t w = (size_t)e->w;
    const double* lv = e->arena + (size_t)s->l * w;
    const double* uv = e->arena + (size_t)s->u * w;
    double* x = e->arena + (size_t)s->v_base * w;
    for (int i = 0; i < s->dim; ++i) {
        double* xi = x + (size_t)i * w;
        for (int k = s->l_row_ptr[i]; k < s->l_row_ptr[i + 1]; ++k) {
            const double* xk = x + (size_t)s->l_col[k] * w;
            const double* lik = lv + (size_t)k * w;
            for (size_t lane = 0; lane < w; ++lane) xi[lane] -= lik[lane] * xk[lane];
        }
    }
    for (int i = s->dim - 1; i >= 0; --i) {
        double* xi = x + (size_t)i * w;
        const int rb = s->u_row_ptr[i];
        for (int k = rb + 1; k < s->u_row_ptr[i + 1]; ++k) {
            const double* xj = x + (size_t)s->u_col[k] * w;
            const double* uij = uv + (size_t)k * w;
            for (size_t lane = 0; lane < w; ++lane) xi[lane] -= uij[lane] * xj[lane];
        }
        const double* diag = uv + (size_t)rb * w;
        for (size_t lane = 0; lane < w; ++lane) xi[lane] /= diag[lane];
    }
}

/* kern::source_value (proj/include/emtgrid/kernels.hpp:68-70) */
static inline double source_value(double mag, double omega, double phase, double t) {
    return omega == 0.0 ? mag : mag * cos(omega * t + phase);
}

/* Engine::run_proc (proj/src/exec.cpp:77-311), one case per KernelId. */
static int run_proc(eng_t* e, const proc_t* p, double t, int step, char* err, int err_len) {
    const emto_schedule* s = e->s;
    const int w = e->w;
    const size_t W = (size_t)w;
    const int* in = s->port_slot + p->in_base;
    const double* sg = s->port_sign + p->in_base;
    const double* par = p->par >= 0 ? e->consts + (size_t)p->par * W : NULL;
    double* st = p->state >= 0 ? e->arena + (size_t)p->state * W : NULL;
    double* A = e->arena;
    switch (p->code) {
    case K_RES: { /* exec.cpp:85-93 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) { g[l] = par[l]; h[l] = 0.0; }
        break;
    }
    case K_IND: { /* exec.cpp:94-103; hist_inductor kernels.hpp:71-73 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            const double vs = rd(e, in[1], l) - rd(e, in[0], l);
            g[l] = par[l];
            h[l] = rd(e, in[2], l) + g[l] * vs;
        }
        break;
    }
    case K_CAP: { /* exec.cpp:104-113; hist_capacitor kernels.hpp:74-76 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            const double vs = rd(e, in[1], l) - rd(e, in[0], l);
            g[l] = par[l];
            h[l] = -rd(e, in[2], l) - g[l] * vs;
        }
        break;
    }
    case K_SRL: { /* exec.cpp:114-123; hist_series_rl kernels.hpp:77-79 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            const double vs = rd(e, in[1], l) - rd(e, in[0], l);
            g[l] = par[l];
            h[l] = par[W + l] * rd(e, in[2], l) + g[l] * vs;
        }
        break;
    }
    case K_VSRC: { /* exec.cpp:124-132 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            g[l] = par[l];
            h[l] = g[l] * source_value(par[W + l], par[2 * W + l], par[3 * W + l], t);
        }
        break;
    }
    case K_ISRC: { /* exec.cpp:133-141 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            g[l] = 0.0;
            h[l] = source_value(par[l], par[W + l], par[2 * W + l], t);
        }
        break;
    }
    case K_CSRC: { /* exec.cpp:142-150 */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            g[l] = 0.0;
            h[l] = par[l] * (p->in_count > 3 ? rd(e, in[3], l) : 0.0);
        }
        break;
    }
    case K_BERG: {
        /* Lossless Bergeron line end (EXTENSION: the reference has no line model,
         * SURVEY.md §0; parity unpinned, checked analytically in tests/test_bergeron.py).
         * Norton form like a current source (g = 0 here; the surge conductance 1/Zc
         * is a parallel resistor stamped by the compiler). With u = vs, i = u/Zc + h
         * at both ends, the travelling-wave relation gives
         *   beta_k(p) = (2/Zc) u_k(t_p) + h_k(t_p)   (pushed into this end's ring)
         *   h_k(t_{p+1}) = -[(1-f) beta_m(p+1-K) + f beta_m(p-K)],  tau = (K+f) dt,
         * beta_m read from the peer end's ring (peer lane / ring slot are constants,
         * so line ends may couple scenario lanes: BASELINE C4 line-split systems).
         * par = [2/Zc, 1-f, f, K, peer_lane, peer_ring_slot]; state = ring[L]. */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        const int L = p->state_len;
        for (int l = 0; l < w; ++l) {
            const double vs = rd(e, in[1], l) - rd(e, in[0], l);
            const double beta = par[l] * vs + h[l];
            st[(size_t)(step % L) * W + (size_t)l] = beta;
        }
        for (int l = 0; l < w; ++l) {
            const int K = (int)par[3 * W + l];
            const size_t pl = (size_t)par[4 * W + l];
            const size_t pr = (size_t)par[5 * W + l];
            int q1 = (step + 1 - K) % L;
            if (q1 < 0) q1 += L;
            const int q0 = q1 == 0 ? L - 1 : q1 - 1;
            const double b1 = A[(pr + (size_t)q1) * W + pl];
            const double b0 = A[(pr + (size_t)q0) * W + pl];
            g[l] = 0.0;
            h[l] = -(par[W + l] * b1 + par[2 * W + l] * b0);
        }
        break;
    }
    case K_SW: { /* exec.cpp:151-165; state [now, changed] */
        double* g = A + (size_t)p->out * W; double* h = A + (size_t)p->out2 * W;
        for (int l = 0; l < w; ++l) {
            int now = par[2 * W + l] != 0.0 ? 1 : 0;
            for (int j = 3; j < p->par_len; ++j)
                if (t >= par[(size_t)j * W + l]) now ^= 1;
            st[W + l] = (double)now != st[l] ? 1.0 : 0.0;
            st[l] = (double)now;
            g[l] = now != 0 ? par[l] : par[W + l];
            h[l] = 0.0;
            if (st[W + l] != 0.0) {
                if (e->events && e->n_events < e->max_events) {
                    e->events[3 * e->n_events + 0] = step;
                    e->events[3 * e->n_events + 1] = l;
                    e->events[3 * e->n_events + 2] = p->id;
                }
                e->n_events++;
            }
        }
        break;
    }
    case K_INJ: { /* exec.cpp:166-174 */
        double* c = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            const double h = rd(e, in[0], l);
            c[l] = h;
            c[W + l] = -h;
        }
        break;
    }
    case K_FACT: { /* exec.cpp:175-204: refactor every lane if any watch slot of any lane is set */
        int refactor = 0;
        for (int k = 0; k < s->nwatch && !refactor; ++k)
            for (int l = 0; l < w && !refactor; ++l)
                if (rd(e, s->watch[k], l) != 0.0) refactor = 1;
        if (!refactor) break;
        for (int k = 0; k < s->nnz; ++k) {
            double* dst = A + (size_t)(s->mat + k) * W;
            for (int l = 0; l < w; ++l) dst[l] = 0.0;
            for (int q = s->ment_ptr[k]; q < s->ment_ptr[k + 1]; ++q) {
                const double* src = A + (size_t)s->ment_slot[q] * W;
                const double sgn = s->ment_sign[q];
                for (int l = 0; l < w; ++l) dst[l] += sgn * src[l];
            }
        }
        int rc = lu_factor(e, err, err_len);
        if (rc != ST_OK) return rc;
        for (int k = 0; k < s->nwatch; ++k) {
            double* cell = A + (size_t)s->watch[k] * W;
            for (int l = 0; l < w; ++l) cell[l] = 0.0;
        }
        double* fc = A + (size_t)s->fcount * W;
        for (int l = 0; l < w; ++l) fc[l] += 1.0;
        break;
    }
    case K_SOLVE: { /* exec.cpp:205-239: gather, lu_solve, finalize, divergence */
        for (int node = 0; node < s->nodes; ++node) {
            double* dst = A + (size_t)(s->v_base + node) * W;
            for (int l = 0; l < w; ++l) dst[l] = 0.0;
            for (int q = s->gat_ptr[node]; q < s->gat_ptr[node + 1]; ++q) {
                const double* src = A + (size_t)s->gat_slot[q] * W;
                for (int l = 0; l < w; ++l) dst[l] += src[l];
            }
        }
        if (s->nodes > 0) lu_solve(e);
        for (int c = 0; c < s->comps; ++c) {
            const int* f = s->fin + 5 * c;
            double* i = A + (size_t)f[0] * W;
            const double* g = A + (size_t)f[1] * W;
            const double* h = A + (size_t)f[2] * W;
            for (int l = 0; l < w; ++l) {
                const double vs = rd(e, f[4], l) - rd(e, f[3], l);
                i[l] = g[l] * vs + h[l];
            }
        }
        for (int node = 0; node < s->nodes; ++node) {
            const double* v = A + (size_t)(s->v_base + node) * W;
            for (int l = 0; l < w; ++l) {
                if (!(fabs(v[l]) <= 1e12)) { /* kDivergenceLimit kernels.hpp:24 */
                    e->err_index = node;
                    e->err_lane = l;
                    return set_err(err, err_len, ST_NONFINITE, "node voltage diverged (at node index %d)", node);
                }
            }
        }
        break;
    }
    case K_GAIN: { /* exec.cpp:240-244 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) o[l] = par[l] * (sg[0] * rd(e, in[0], l));
        break;
    }
    case K_SUM: { /* exec.cpp:245-253: signs applied before sequential accumulation */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            double acc = 0.0;
            for (int j = 0; j < p->in_count; ++j) acc += sg[j] * rd(e, in[j], l);
            o[l] = acc;
        }
        break;
    }
    case K_INTEG: { /* exec.cpp:254-264; ctl_integrate kernels.hpp:80-82 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            const double u = sg[0] * rd(e, in[0], l);
            const double y = st[l] + par[l] * (u + st[W + l]);
            st[l] = y;
            st[W + l] = u;
            o[l] = y;
        }
        break;
    }
    case K_LAG: { /* exec.cpp:265-275; ctl_lag kernels.hpp:83-85 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            const double u = sg[0] * rd(e, in[0], l);
            const double y = par[l] * st[l] + par[W + l] * (u + st[W + l]);
            st[l] = y;
            st[W + l] = u;
            o[l] = y;
        }
        break;
    }
    case K_LIM: { /* exec.cpp:276-282; ctl_clamp kernels.hpp:86-88 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            const double u = sg[0] * rd(e, in[0], l);
            const double lo = par[l], hi = par[W + l];
            o[l] = u < lo ? lo : (u > hi ? hi : u);
        }
        break;
    }
    case K_PI: { /* exec.cpp:283-292 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) {
            const double u = sg[0] * rd(e, in[0], l);
            st[l] = st[l] + par[W + l] * (u + st[W + l]);
            st[W + l] = u;
            o[l] = par[l] * u + st[l];
        }
        break;
    }
    case K_CMP: { /* exec.cpp:293-298 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) o[l] = sg[0] * rd(e, in[0], l) >= sg[1] * rd(e, in[1], l) ? 1.0 : 0.0;
        break;
    }
    case K_CONST: { /* exec.cpp:299-303 */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) o[l] = par[l];
        break;
    }
    case K_DELAY: { /* exec.cpp:304-308: input is a latched shadow slot */
        double* o = A + (size_t)p->out * W;
        for (int l = 0; l < w; ++l) o[l] = sg[0] * rd(e, in[0], l);
        break;
    }
    default:
        return set_err(err, err_len, ST_UNKNOWN_KIND, "kernel code %d is not registered", p->code);
    }
    return ST_OK;
}

int emto_interpret(const emto_schedule* s, const double* initial, int64_t initial_len, int steps,
                   double* waves, double* time, int* factor_count, double* final_arena,
                   int32_t* events, int max_events, int* n_events, int* err_index, int* err_lane,
                   int* err_step, char* err, int err_len) {
    /* validate_initial (exec.cpp:340-348) */
    if (initial_len != (int64_t)s->extent * s->width)
        return set_err(err, err_len, ST_DIMENSION, "initial state size %lld does not match extent %d x width %d",
                       (long long)initial_len, s->extent, s->width);
    /* decode (exec.cpp:31-62): unknown kernel codes are rejected up front */
    for (int k = 0; k < s->nproc; ++k)
        if (s->procs[k].code < 0 || s->procs[k].code >= K_COUNT)
            return set_err(err, err_len, ST_UNKNOWN_KIND, "kernel code %d is not registered (at process %d)",
                           s->procs[k].code, s->procs[k].id);
    /* LU fill consistency (exec.cpp:353-357) */
    if (s->l_row_ptr[s->dim] != s->l_nnz || s->u_row_ptr[s->dim] != s->u_nnz)
        return set_err(err, err_len, ST_MALFORMED, "schedule LU fill sizes are inconsistent");

    eng_t e;
    memset(&e, 0, sizeof e);
    e.s = s;
    e.w = s->width;
    e.consts = s->const_table;
    e.arena = (double*)malloc(sizeof(double) * (size_t)(initial_len + 1));
    memcpy(e.arena, initial, sizeof(double) * (size_t)initial_len);
    e.events = events;
    e.max_events = max_events;
    e.err_index = e.err_lane = -1;
    const size_t cols = (size_t)s->nch * (size_t)s->width;
    int rc = ST_OK;
    int step = 0;
    for (step = 0; step < steps && rc == ST_OK; ++step) {
        const double t = (double)(step + 1) * s->dt; /* exec.cpp:366 */
        for (int layer = 0; layer < s->layers && rc == ST_OK; ++layer)
            for (int k = s->layer_begin[layer]; k < s->layer_begin[layer + 1] && rc == ST_OK; ++k)
                rc = run_proc(&e, &s->procs[k], t, step, err, err_len);
        if (rc != ST_OK) break;
        /* record (exec.cpp:313-321) then latch (exec.cpp:323-329) */
        if (time) time[step] = t;
        if (waves)
            for (int ch = 0; ch < s->nch; ++ch)
                for (int l = 0; l < s->width; ++l)
                    waves[(size_t)step * cols + (size_t)ch * (size_t)s->width + (size_t)l] = rd(&e, s->ch_slot[ch], l);
        for (int q = 0; q < s->nlatch; ++q) {
            double* dst = e.arena + (size_t)s->latch_shadow[q] * (size_t)s->width;
            const double* src = e.arena + (size_t)s->latch_live[q] * (size_t)s->width;
            for (int l = 0; l < s->width; ++l) dst[l] = src[l];
        }
    }
    if (err_index) *err_index = e.err_index;
    if (err_lane) *err_lane = e.err_lane;
    if (err_step) *err_step = rc == ST_OK ? -1 : step;
    if (n_events) *n_events = e.n_events;
    /* ExecStats::factor_count = lane 0 fcount (exec.cpp:376) */
    if (factor_count) *factor_count = (int)rd(&e, s->fcount, 0);
    if (final_arena) memcpy(final_arena, e.arena, sizeof(double) * (size_t)initial_len);
    free(e.arena);
    return rc;
}
