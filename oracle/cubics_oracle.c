/*
 * cubics_oracle.c - TEST INFRASTRUCTURE ONLY (see cubics_oracle.h).
 *
 * Plain-C restatement of the reference hot path. Every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj). Data layout follows the
 * reference Domain: u64 words, bit i = value offset + i (include/fd/domain.hpp:21-78).
 * Integer semantics follow the compiled reference, including __int128 comparisons and the
 * checked int64 arithmetic of the linear propagator.
 */
#include "cubics_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ---------------------------------------------------------------- model view */
typedef struct {
    int n;
    const int64_t* off;
    const int32_t* width;
    int32_t* ws; /* word start per var, n+1 entries */
    int total;   /* total u64 words */
    const cubics_model_desc* d;
} Model;

static int model_init(Model* m, const cubics_model_desc* d) {
    m->d = d;
    m->n = d->n_vars;
    m->off = d->var_offset;
    m->width = d->var_width;
    m->ws = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m->n + 1));
    if (!m->ws) return CUBICS_E_INVALID;
    int acc = 0;
    for (int v = 0; v < m->n; ++v) {
        m->ws[v] = acc;
        acc += (m->width[v] + 63) / 64;
    }
    m->ws[m->n] = acc;
    m->total = acc;
    return CUBICS_OK;
}

static void model_free(Model* m) { free(m->ws); }

static void init_words(const Model* m, uint64_t* w) {
    if (m->d->var_words) {
        memcpy(w, m->d->var_words, sizeof(uint64_t) * (size_t)m->total);
        return;
    }
    memset(w, 0, sizeof(uint64_t) * (size_t)m->total);
    for (int v = 0; v < m->n; ++v)
        for (int i = 0; i < m->width[v]; ++i) w[m->ws[v] + i / 64] |= (uint64_t)1 << (i % 64);
}

/* ---------------------------------------------------------------- domain queries
 * (domain.cpp:10-163: contains, size/min/max caches recomputed from the words) */
static int d_nw(const Model* m, int v) { return m->ws[v + 1] - m->ws[v]; }

static int d_size(const Model* m, const uint64_t* W, int v) {
    int s = 0;
    for (int i = m->ws[v]; i < m->ws[v + 1]; ++i) s += __builtin_popcountll(W[i]);
    return s;
}

static int64_t d_min(const Model* m, const uint64_t* W, int v) { /* domain.cpp:504-525 */
    for (int i = 0; i < d_nw(m, v); ++i) {
        uint64_t x = W[m->ws[v] + i];
        if (x) return m->off[v] + i * 64 + __builtin_ctzll(x);
    }
    return m->off[v];
}

static int64_t d_max(const Model* m, const uint64_t* W, int v) {
    for (int i = d_nw(m, v) - 1; i >= 0; --i) {
        uint64_t x = W[m->ws[v] + i];
        if (x) return m->off[v] + i * 64 + 63 - __builtin_clzll(x);
    }
    return m->off[v];
}

static int d_contains(const Model* m, const uint64_t* W, int v, i128 x) { /* domain.cpp:390-395 */
    if (x < (i128)m->off[v] || x >= (i128)m->off[v] + m->width[v]) return 0;
    int pos = (int)(x - m->off[v]);
    return (int)((W[m->ws[v] + pos / 64] >> (pos % 64)) & 1);
}

/* RemovalSet::add_value / add_range / add_all (propagation.cpp:42-63): only values present in
 * the snapshot are recorded; the set is a dense mask array (union-merge is order-free). */
static void add_value(const Model* m, const uint64_t* S, uint64_t* R, int v, i128 x) {
    if (!d_contains(m, S, v, x)) return;
    int pos = (int)(x - m->off[v]);
    R[m->ws[v] + pos / 64] |= (uint64_t)1 << (pos % 64);
}

static void add_range(const Model* m, const uint64_t* S, uint64_t* R, int v, int64_t lo, int64_t hi) {
    if (d_size(m, S, v) == 0) return;
    int64_t mn = d_min(m, S, v), mx = d_max(m, S, v);
    if (lo < mn) lo = mn;
    if (hi > mx) hi = mx;
    for (int64_t x = lo; x <= hi; ++x) add_value(m, S, R, v, x);
}

/* wrapping int64 add, as the compiled reference computes `lit + 1` / `lit - 1` */
static int64_t wrap_add(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }

/* ---------------------------------------------------------------- propagators */

/* prop_rel_bin (propagation.cpp:120-194) */
static void prop_rel_bin(const Model* m, int c, const uint64_t* S, uint64_t* R) {
    const cubics_model_desc* d = m->d;
    int t0 = d->con_start[c];
    int x = d->term_var[t0];
    int op = d->con_op[c];
    int64_t k64 = d->con_value[c];
    if (d_size(m, S, x) == 0) return;
    int64_t xmin = d_min(m, S, x), xmax = d_max(m, S, x);
    if (d->con_start[c + 1] - t0 == 1) { /* literal form :126-141 */
        int64_t lit = k64;
        switch (op) {
        case CUBICS_LT: add_range(m, S, R, x, lit, xmax); break;
        case CUBICS_LE: add_range(m, S, R, x, wrap_add(lit, 1), xmax); break;
        case CUBICS_GT: add_range(m, S, R, x, xmin, lit); break;
        case CUBICS_GE: add_range(m, S, R, x, xmin, wrap_add(lit, -1)); break;
        case CUBICS_EQ:
            for (int64_t v = xmin; v <= xmax; ++v)
                if (d_contains(m, S, x, v) && v != lit) add_value(m, S, R, x, v);
            break;
        case CUBICS_NE: add_value(m, S, R, x, lit); break;
        }
        return;
    }
    int y = d->term_var[t0 + 1];
    if (d_size(m, S, y) == 0) return;
    int64_t ymin = d_min(m, S, y), ymax = d_max(m, S, y);
    i128 k = k64;
    /* keep_x / keep_y (:148-157): remove every present value failing the predicate */
    for (int64_t v = xmin; v <= xmax; ++v) {
        if (!d_contains(m, S, x, v)) continue;
        i128 V = v;
        int keep = 1;
        switch (op) {
        case CUBICS_LT: keep = V < (i128)ymax + k; break;
        case CUBICS_LE: keep = V <= (i128)ymax + k; break;
        case CUBICS_GT: keep = V > (i128)ymin + k; break;
        case CUBICS_GE: keep = V >= (i128)ymin + k; break;
        case CUBICS_EQ: keep = d_contains(m, S, y, V - k); break; /* fits_i64 implied by range */
        case CUBICS_NE: keep = 1; break;
        }
        if (!keep) add_value(m, S, R, x, V);
    }
    for (int64_t w = ymin; w <= ymax; ++w) {
        if (!d_contains(m, S, y, w)) continue;
        i128 Wv = w;
        int keep = 1;
        switch (op) {
        case CUBICS_LT: keep = (i128)xmin < Wv + k; break;
        case CUBICS_LE: keep = (i128)xmin <= Wv + k; break;
        case CUBICS_GT: keep = (i128)xmax > Wv + k; break;
        case CUBICS_GE: keep = (i128)xmax >= Wv + k; break;
        case CUBICS_EQ: keep = d_contains(m, S, x, Wv + k); break;
        case CUBICS_NE: keep = 1; break;
        }
        if (!keep) add_value(m, S, R, y, Wv);
    }
    if (op == CUBICS_NE) { /* :180-191 */
        if (d_size(m, S, y) == 1) add_value(m, S, R, x, (i128)ymin + k);
        if (d_size(m, S, x) == 1) add_value(m, S, R, y, (i128)xmin - k);
    }
}

/* checked_mul / checked_add (propagation.cpp:198-210) */
static int64_t checked_mul(int64_t a, int64_t b, int* ovf) {
    int64_t r;
    if (__builtin_mul_overflow(a, b, &r)) *ovf = 1;
    return r;
}
static int64_t checked_add(int64_t a, int64_t b, int* ovf) {
    int64_t r;
    if (__builtin_add_overflow(a, b, &r)) *ovf = 1;
    return r;
}

/* filter_linear_le (propagation.cpp:213-236). Returns nonzero on overflow. */
static int filter_linear_le(const Model* m, int nt, const int32_t* var, const int64_t* coeff,
                            int64_t bound, const uint64_t* S, uint64_t* R) {
    int64_t tmin_stack[64];
    int64_t* tmin = nt <= 64 ? tmin_stack : (int64_t*)malloc(sizeof(int64_t) * (size_t)nt);
    int ovf = 0;
    int64_t total = 0;
    for (int i = 0; i < nt; ++i) {
        int v = var[i];
        if (d_size(m, S, v) == 0) goto done;
        tmin[i] = coeff[i] > 0 ? checked_mul(coeff[i], d_min(m, S, v), &ovf)
                               : checked_mul(coeff[i], d_max(m, S, v), &ovf);
        if (ovf) goto done;
        total = checked_add(total, tmin[i], &ovf);
        if (ovf) goto done;
    }
    for (int j = 0; j < nt; ++j) {
        int v = var[j];
        int64_t rest = checked_add(total, (int64_t)(0 - (uint64_t)tmin[j]), &ovf);
        if (ovf) goto done;
        i128 budget = (i128)bound - (i128)rest;
        i128 a = coeff[j];
        int64_t mn = d_min(m, S, v), mx = d_max(m, S, v);
        for (int64_t x = mn; x <= mx; ++x)
            if (d_contains(m, S, v, x) && a * (i128)x > budget) add_value(m, S, R, v, x);
    }
done:
    if (tmin != tmin_stack) free(tmin);
    return ovf;
}

/* prop_linear (propagation.cpp:240-252) */
static int prop_linear(const Model* m, int c, const uint64_t* S, uint64_t* R) {
    const cubics_model_desc* d = m->d;
    int t0 = d->con_start[c], nt = d->con_start[c + 1] - t0;
    if (filter_linear_le(m, nt, d->term_var + t0, d->term_coeff + t0, d->con_value[c], S, R)) return 1;
    if (d->con_op[c] == CUBICS_LIN_EQ) {
        int ovf = 0;
        int64_t* neg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nt ? nt : 1));
        for (int i = 0; i < nt; ++i) neg[i] = checked_mul(d->term_coeff[t0 + i], -1, &ovf);
        int64_t nb = checked_mul(d->con_value[c], -1, &ovf);
        if (!ovf) ovf = filter_linear_le(m, nt, d->term_var + t0, neg, nb, S, R);
        free(neg);
        return ovf;
    }
    return 0;
}

/* prop_alldiff_fc (propagation.cpp:254-268) */
static void prop_alldiff_fc(const Model* m, int c, const uint64_t* S, uint64_t* R) {
    const cubics_model_desc* d = m->d;
    int t0 = d->con_start[c], nt = d->con_start[c + 1] - t0;
    for (int i = 0; i < nt; ++i) {
        int vi = d->term_var[t0 + i];
        if (d_size(m, S, vi) != 1) continue;
        int64_t val = d_min(m, S, vi);
        for (int j = 0; j < nt; ++j)
            if (j != i) add_value(m, S, R, d->term_var[t0 + j], val);
    }
}

/* ---- prop_alldiff_gac (propagation.cpp:270-433): Kuhn matching in member order, residual
 * graph, SCCs, reachability from free values. */
typedef struct {
    int n, mv;           /* members, distinct values */
    int64_t* value_of;   /* value index -> value (sorted) */
    int* adj_start;      /* member -> value indices (ascending) */
    int* adj;
    int* match_var;
    int* match_val;
    char* visited;
} Gac;

static int try_augment(Gac* g, int var) { /* AlldiffGraph::try_augment :284-296 */
    for (int e = g->adj_start[var]; e < g->adj_start[var + 1]; ++e) {
        int j = g->adj[e];
        if (g->visited[j]) continue;
        g->visited[j] = 1;
        if (g->match_val[j] < 0 || try_augment(g, g->match_val[j])) {
            g->match_var[var] = j;
            g->match_val[j] = var;
            return 1;
        }
    }
    return 0;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

/* Tarjan SCC over the residual graph (restates tarjan_scc :299-344, recursive form). */
typedef struct {
    int total;
    const int* ostart;
    const int* oadj;
    int *index, *low, *stack, *on, *comp;
    int sp, next_index, next_comp;
} Scc;

static void scc_visit(Scc* s, int u) {
    s->index[u] = s->low[u] = s->next_index++;
    s->stack[s->sp++] = u;
    s->on[u] = 1;
    for (int e = s->ostart[u]; e < s->ostart[u + 1]; ++e) {
        int v = s->oadj[e];
        if (s->index[v] < 0) {
            scc_visit(s, v);
            if (s->low[v] < s->low[u]) s->low[u] = s->low[v];
        } else if (s->on[v] && s->index[v] < s->low[u]) {
            s->low[u] = s->index[v];
        }
    }
    if (s->low[u] == s->index[u]) {
        for (;;) {
            int w = s->stack[--s->sp];
            s->on[w] = 0;
            s->comp[w] = s->next_comp;
            if (w == u) break;
        }
        s->next_comp++;
    }
}

static void prop_alldiff_gac(const Model* m, int c, const uint64_t* S, uint64_t* R) {
    const cubics_model_desc* d = m->d;
    int t0 = d->con_start[c], n = d->con_start[c + 1] - t0;
    const int32_t* vars = d->term_var + t0;
    /* universe = sorted unique member values (:353-360) */
    int cap = 0;
    for (int i = 0; i < n; ++i) cap += d_size(m, S, vars[i]);
    Gac g;
    memset(&g, 0, sizeof g);
    g.n = n;
    int64_t* uni = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap + 1));
    int u = 0;
    for (int i = 0; i < n; ++i) {
        int v = vars[i];
        int64_t mn = d_min(m, S, v), mx = d_max(m, S, v);
        if (d_size(m, S, v) == 0) continue;
        for (int64_t x = mn; x <= mx; ++x)
            if (d_contains(m, S, v, x)) uni[u++] = x;
    }
    qsort(uni, (size_t)u, sizeof(int64_t), cmp_i64);
    int mv = 0;
    for (int i = 0; i < u; ++i)
        if (mv == 0 || uni[i] != uni[mv - 1]) uni[mv++] = uni[i];
    g.mv = mv;
    g.value_of = uni;
    g.adj_start = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    g.adj = (int*)malloc(sizeof(int) * (size_t)(cap + 1));
    int e = 0;
    for (int i = 0; i < n; ++i) { /* var_values (:367-370), ascending */
        g.adj_start[i] = e;
        int v = vars[i];
        int j = 0;
        for (int64_t x = d_min(m, S, v); d_size(m, S, v) && x <= d_max(m, S, v); ++x) {
            if (!d_contains(m, S, v, x)) continue;
            while (uni[j] < x) ++j;
            g.adj[e++] = j;
        }
    }
    g.adj_start[n] = e;
    g.match_var = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    g.match_val = (int*)malloc(sizeof(int) * (size_t)(mv + 1));
    g.visited = (char*)malloc((size_t)(mv + 1));
    for (int i = 0; i < n; ++i) g.match_var[i] = -1;
    for (int j = 0; j < mv; ++j) g.match_val[j] = -1;
    for (int i = 0; i < n; ++i) { /* :374-377 */
        memset(g.visited, 0, (size_t)(mv + 1));
        try_augment(&g, i);
    }
    int total = n + mv;
    int* ostart = NULL;
    int* oadj = NULL;
    int* idx = NULL;
    char* reached = NULL;
    int* queue = NULL;
    Scc s;
    memset(&s, 0, sizeof s);
    for (int i = 0; i < n; ++i) {
        if (g.match_var[i] < 0) { /* :379-386: wipe the first unmatched member */
            int v = vars[i];
            if (d_size(m, S, v)) add_range(m, S, R, v, d_min(m, S, v), d_max(m, S, v));
            goto out;
        }
    }
    /* residual orientation (:388-397): matched var -> value, others value -> var */
    ostart = (int*)calloc((size_t)(total + 1), sizeof(int));
    oadj = (int*)malloc(sizeof(int) * (size_t)(e + 1));
    for (int i = 0; i < n; ++i)
        for (int q = g.adj_start[i]; q < g.adj_start[i + 1]; ++q) {
            int j = g.adj[q];
            if (g.match_var[i] == j) ostart[i + 1]++;
            else ostart[n + j + 1]++;
        }
    for (int k = 0; k < total; ++k) ostart[k + 1] += ostart[k];
    idx = (int*)malloc(sizeof(int) * (size_t)(total + 1));
    for (int k = 0; k < total; ++k) idx[k] = ostart[k];
    for (int i = 0; i < n; ++i)
        for (int q = g.adj_start[i]; q < g.adj_start[i + 1]; ++q) {
            int j = g.adj[q];
            if (g.match_var[i] == j) oadj[idx[i]++] = n + j;
            else oadj[idx[n + j]++] = i;
        }
    s.total = total;
    s.ostart = ostart;
    s.oadj = oadj;
    s.index = (int*)malloc(sizeof(int) * (size_t)total);
    s.low = (int*)malloc(sizeof(int) * (size_t)total);
    s.stack = (int*)malloc(sizeof(int) * (size_t)total);
    s.on = (int*)calloc((size_t)total, sizeof(int));
    s.comp = (int*)malloc(sizeof(int) * (size_t)total);
    for (int k = 0; k < total; ++k) s.index[k] = -1;
    for (int k = 0; k < total; ++k)
        if (s.index[k] < 0) scc_visit(&s, k);
    /* reachability from unmatched values (:402-418) */
    reached = (char*)calloc((size_t)total, 1);
    queue = (int*)malloc(sizeof(int) * (size_t)total);
    int qn = 0;
    for (int j = 0; j < mv; ++j)
        if (g.match_val[j] < 0) {
            reached[n + j] = 1;
            queue[qn++] = n + j;
        }
    while (qn) {
        int a = queue[--qn];
        for (int q = ostart[a]; q < ostart[a + 1]; ++q) {
            int b = oadj[q];
            if (!reached[b]) {
                reached[b] = 1;
                queue[qn++] = b;
            }
        }
    }
    for (int i = 0; i < n; ++i) /* :420-431 */
        for (int q = g.adj_start[i]; q < g.adj_start[i + 1]; ++q) {
            int j = g.adj[q];
            if (g.match_var[i] == j) continue;
            if (s.comp[i] == s.comp[n + j]) continue;
            if (reached[n + j]) continue;
            add_value(m, S, R, vars[i], g.value_of[j]);
        }
out:
    free(uni);
    free(g.adj_start);
    free(g.adj);
    free(g.match_var);
    free(g.match_val);
    free(g.visited);
    free(ostart);
    free(oadj);
    free(idx);
    free(s.index);
    free(s.low);
    free(s.stack);
    free(s.on);
    free(s.comp);
    free(reached);
    free(queue);
}

/* Extension (no reference counterpart, BASELINE config 5): positive table constraint. A value is
 * supported when some allowed tuple has it in its position and every other component in the
 * respective domain (positions are independent, as Linear treats repeated variables). */
static void prop_table(const Model* m, int c, const uint64_t* S, uint64_t* R) {
    const cubics_model_desc* d = m->d;
    const int t0 = d->con_start[c], k = d->con_start[c + 1] - t0;
    const int64_t nt = d->con_value[c];
    const int64_t* data = d->table_data + d->table_start[c];
    for (int j = 0; j < k; ++j)
        if (d_size(m, S, d->term_var[t0 + j]) == 0) return;
    uint64_t* sup = (uint64_t*)calloc((size_t)k * 16u, sizeof(uint64_t));
    for (int64_t i = 0; i < nt; ++i) {
        int valid = 1;
        for (int j = 0; j < k && valid; ++j) valid = d_contains(m, S, d->term_var[t0 + j], data[i * k + j]);
        if (!valid) continue;
        for (int j = 0; j < k; ++j) {
            int pos = (int)(data[i * k + j] - m->off[d->term_var[t0 + j]]);
            sup[j * 16 + pos / 64] |= (uint64_t)1 << (pos % 64);
        }
    }
    for (int j = 0; j < k; ++j) {
        int v = d->term_var[t0 + j];
        for (int w = 0; w < d_nw(m, v); ++w) R[m->ws[v] + w] |= S[m->ws[v] + w] & ~sup[j * 16 + w];
    }
    free(sup);
}

/* propagate_one (propagation.cpp:435-442). Returns nonzero on overflow. */
static int propagate_one(const Model* m, int c, const uint64_t* S, uint64_t* R, int alldiff) {
    switch (m->d->con_kind[c]) {
    case CUBICS_RELBIN: prop_rel_bin(m, c, S, R); return 0;
    case CUBICS_LINEAR: return prop_linear(m, c, S, R);
    case CUBICS_TABLE: prop_table(m, c, S, R); return 0;
    default:
        if (alldiff == CUBICS_ARC_CONSISTENT) prop_alldiff_gac(m, c, S, R);
        else prop_alldiff_fc(m, c, S, R);
        return 0;
    }
}

/* ---------------------------------------------------------------- trail (state.cpp:9-44) */
typedef struct {
    int var, level, prev_top;
    size_t at; /* offset into words */
} TrailEntry;

typedef struct {
    const Model* m;
    uint64_t* W; /* current domains */
    int level;
    int* top;    /* per var: level of its newest saved entry, -1 = none */
    TrailEntry* e;
    size_t ne, cap;
    uint64_t* saved;
    size_t nsaved, scap;
} Store;

static void store_save(Store* s, int var) { /* save_on_modify :12-17 */
    if (s->top[var] == s->level) return;
    const Model* m = s->m;
    int nw = d_nw(m, var);
    if (s->ne == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 256;
        s->e = (TrailEntry*)realloc(s->e, sizeof(TrailEntry) * s->cap);
    }
    if (s->nsaved + (size_t)nw > s->scap) {
        s->scap = 2 * (s->scap + (size_t)nw) + 256;
        s->saved = (uint64_t*)realloc(s->saved, sizeof(uint64_t) * s->scap);
    }
    memcpy(s->saved + s->nsaved, s->W + m->ws[var], sizeof(uint64_t) * (size_t)nw);
    s->e[s->ne].var = var;
    s->e[s->ne].level = s->level;
    s->e[s->ne].prev_top = s->top[var];
    s->e[s->ne].at = s->nsaved;
    s->ne++;
    s->nsaved += (size_t)nw;
    s->top[var] = s->level;
}

static void store_pop_level(Store* s) { /* pop_level + restore_to_level :19-44 */
    int target = s->level - 1;
    const Model* m = s->m;
    while (s->ne && s->e[s->ne - 1].level > target) {
        TrailEntry* t = &s->e[--s->ne];
        memcpy(s->W + m->ws[t->var], s->saved + t->at, sizeof(uint64_t) * (size_t)d_nw(m, t->var));
        s->top[t->var] = t->prev_top;
        s->nsaved = t->at;
    }
    s->level = target;
}

/* ---------------------------------------------------------------- round / fixpoint */
typedef struct {
    uint64_t* snap;
    uint64_t* rm;
} Scratch;

/* propagate_round (propagation.cpp:480-514). status: 0 Changed 1 Stable 2 Failed; -1 overflow */
static int propagate_round(const Model* m, uint64_t* W, int alldiff, Scratch* sc, Store* st,
                           int* failed_var) {
    size_t bytes = sizeof(uint64_t) * (size_t)m->total;
    memcpy(sc->snap, W, bytes);
    memset(sc->rm, 0, bytes);
    for (int c = 0; c < m->d->n_cons; ++c)
        if (propagate_one(m, c, sc->snap, sc->rm, alldiff)) return -1;
    int changed = 0;
    for (int v = 0; v < m->n; ++v) {
        int would = 0;
        for (int i = m->ws[v]; i < m->ws[v + 1]; ++i)
            if (W[i] & sc->rm[i]) would = 1;
        if (!would) continue;
        if (st) store_save(st, v);
        for (int i = m->ws[v]; i < m->ws[v + 1]; ++i) W[i] &= ~sc->rm[i];
        changed = 1;
    }
    if (changed) {
        for (int v = 0; v < m->n; ++v)
            if (d_size(m, W, v) == 0) {
                *failed_var = v;
                return 2;
            }
        return 0;
    }
    return 1;
}

/* propagate_fixpoint (propagation.cpp:516-532); max_rounds > 0 caps the loop. */
static int fixpoint(const Model* m, uint64_t* W, int alldiff, int max_rounds, Scratch* sc, Store* st,
                    cubics_fixpoint_result* out) {
    out->failed = 0;
    out->failed_var = -1;
    out->rounds = 0;
    out->last_status = 1;
    for (;;) {
        int fv = -1;
        int r = propagate_round(m, W, alldiff, sc, st, &fv);
        if (r < 0) return CUBICS_E_OVERFLOW;
        out->rounds++;
        out->last_status = r;
        if (r == 2) {
            out->failed = 1;
            out->failed_var = fv;
            return CUBICS_OK;
        }
        if (r == 1) return CUBICS_OK;
        if (max_rounds > 0 && out->rounds >= max_rounds) return CUBICS_OK;
    }
}

/* ---------------------------------------------------------------- DFS (search.cpp:56-170) */
typedef struct {
    const Model* m;
    const cubics_search_config* cfg;
    Store st;
    Scratch sc;
    cubics_stats stats;
    int optimizing, minimizing, obj;
    int has_bound;
    int64_t bound;
    int64_t* values;
    int64_t* best;
    int has_best;
    cubics_solution_cb cb;
    void* user;
    int limit_hit, user_stop, error;
} Dfs;

static int select_variable(const Dfs* s) { /* search.cpp:13-28 */
    const Model* m = s->m;
    int best = -1, best_size = 0;
    for (int v = 0; v < m->n; ++v) {
        int sz = d_size(m, s->st.W, v);
        if (sz <= 1) continue;
        if (s->cfg->var_heuristic == CUBICS_INPUT_ORDER) return v;
        if (best < 0 || sz < best_size) {
            best = v;
            best_size = sz;
        }
    }
    return best;
}

static int emit_solution(Dfs* s) { /* search.cpp:134-156 */
    const Model* m = s->m;
    for (int v = 0; v < m->n; ++v) s->values[v] = d_min(m, s->st.W, v);
    s->stats.solutions++;
    if (s->optimizing) {
        memcpy(s->best, s->values, sizeof(int64_t) * (size_t)m->n);
        s->has_best = 1;
        s->bound = s->values[s->obj];
        s->has_bound = 1;
    }
    if (s->cb && !s->cb(s->user, s->values, m->n)) {
        s->user_stop = 1;
        return 0;
    }
    if (s->stats.solutions >= s->cfg->max_solutions) {
        s->user_stop = 1;
        return 0;
    }
    return 1;
}

static void remove_value(const Model* m, uint64_t* W, int v, int64_t x) {
    int pos = (int)(x - m->off[v]);
    W[m->ws[v] + pos / 64] &= ~((uint64_t)1 << (pos % 64));
}

static int descend(Dfs* s) { /* search.cpp:80-132 */
    const Model* m = s->m;
    uint64_t* W = s->st.W;
    ++s->stats.nodes;
    if (s->cfg->node_limit && s->stats.nodes > s->cfg->node_limit) {
        s->limit_hit = 1;
        return 0;
    }
    if (s->optimizing && s->has_bound) { /* :87-101 */
        int o = s->obj;
        int shrink = s->minimizing ? d_max(m, W, o) >= s->bound : d_min(m, W, o) <= s->bound;
        if (shrink) {
            store_save(&s->st, o);
            /* remove_above(bound-1) / remove_below(bound+1) (domain.cpp:406-440) */
            for (int i = 0; i < m->width[o]; ++i) {
                int64_t x = m->off[o] + i;
                if (s->minimizing ? x > s->bound - 1 : x < s->bound + 1) remove_value(m, W, o, x);
            }
            if (d_size(m, W, o) == 0) {
                ++s->stats.failures;
                return 1;
            }
        }
    }
    cubics_fixpoint_result fx;
    int rc = fixpoint(m, W, s->cfg->alldiff, 0, &s->sc, &s->st, &fx);
    if (rc != CUBICS_OK) {
        s->error = rc;
        return 0;
    }
    s->stats.rounds += (uint64_t)fx.rounds;
    if (fx.failed) {
        ++s->stats.failures;
        return 1;
    }
    int var = select_variable(s);
    if (var < 0) return emit_solution(s);
    int64_t val = d_min(m, W, var); /* select_value :30-32 */

    s->st.level++; /* push_level; save; assign; descend; pop_level (:118-124) */
    store_save(&s->st, var);
    for (int i = m->ws[var]; i < m->ws[var + 1]; ++i) W[i] = 0;
    {
        int pos = (int)(val - m->off[var]);
        W[m->ws[var] + pos / 64] |= (uint64_t)1 << (pos % 64);
    }
    int keep = descend(s);
    store_pop_level(&s->st);
    if (!keep) return 0;

    s->st.level++; /* push_level; save; remove; descend; pop_level (:126-131) */
    store_save(&s->st, var);
    remove_value(m, W, var, val);
    keep = descend(s);
    store_pop_level(&s->st);
    return keep;
}

static int run_dfs(const cubics_model_desc* d, const cubics_search_config* cfg, cubics_solution_cb cb,
                   void* user, int64_t* best_values, cubics_result* out, int optimize_call) {
    if (!d || !cfg || !out) return CUBICS_E_INVALID;
    memset(out, 0, sizeof *out);
    Model m;
    if (model_init(&m, d)) return CUBICS_E_INVALID;
    int optimizing = d->goal != CUBICS_SATISFY;
    if (optimize_call && !optimizing) {
        model_free(&m);
        return CUBICS_E_NO_OBJECTIVE;
    }
    Dfs s;
    memset(&s, 0, sizeof s);
    s.m = &m;
    s.cfg = cfg;
    s.optimizing = optimizing;
    s.minimizing = d->goal == CUBICS_MINIMIZE;
    s.obj = d->goal_var;
    s.cb = cb;
    s.user = user;
    s.has_bound = cfg->has_initial_bound != 0; /* Dfs::set_initial_bound (search.cpp:63) */
    s.bound = cfg->initial_bound;
    size_t bytes = sizeof(uint64_t) * (size_t)(m.total + 1);
    s.st.m = &m;
    s.st.W = (uint64_t*)malloc(bytes);
    s.st.top = (int*)malloc(sizeof(int) * (size_t)(m.n + 1));
    for (int v = 0; v < m.n; ++v) s.st.top[v] = -1;
    s.sc.snap = (uint64_t*)malloc(bytes);
    s.sc.rm = (uint64_t*)malloc(bytes);
    s.values = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m.n + 1));
    s.best = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m.n + 1));
    init_words(&m, s.st.W);
    descend(&s);
    out->stats = s.stats;
    out->engine = CUBICS_ENGINE_PARITY;
    out->contexts = 1;
    if (optimize_call) {
        out->complete = !s.limit_hit;
        out->has_solution = s.has_best;
        if (s.has_best) {
            out->objective = s.best[s.obj];
            if (best_values) memcpy(best_values, s.best, sizeof(int64_t) * (size_t)m.n);
        }
    } else {
        out->complete = !s.limit_hit && !s.user_stop;
        out->has_solution = s.stats.solutions > 0;
    }
    int rc = s.error;
    free(s.st.W);
    free(s.st.top);
    free(s.st.e);
    free(s.st.saved);
    free(s.sc.snap);
    free(s.sc.rm);
    free(s.values);
    free(s.best);
    model_free(&m);
    return rc;
}

int oracle_solve_satisfy(const cubics_model_desc* d, const cubics_search_config* cfg,
                         cubics_solution_cb cb, void* user, cubics_result* out) {
    return run_dfs(d, cfg, cb, user, NULL, out, 0);
}

int oracle_solve_optimize(const cubics_model_desc* d, const cubics_search_config* cfg,
                          int64_t* best_values, cubics_result* out) {
    return run_dfs(d, cfg, NULL, NULL, best_values, out, 1);
}

int oracle_propagate(const cubics_model_desc* d, uint64_t* words, int32_t alldiff, int32_t max_rounds,
                     cubics_fixpoint_result* out) {
    if (!d || !words || !out) return CUBICS_E_INVALID;
    Model m;
    if (model_init(&m, d)) return CUBICS_E_INVALID;
    Scratch sc;
    size_t bytes = sizeof(uint64_t) * (size_t)(m.total + 1);
    sc.snap = (uint64_t*)malloc(bytes);
    sc.rm = (uint64_t*)malloc(bytes);
    int rc = fixpoint(&m, words, alldiff, max_rounds, &sc, NULL, out);
    free(sc.snap);
    free(sc.rm);
    model_free(&m);
    return rc;
}

int oracle_removals(const cubics_model_desc* d, const uint64_t* words, int32_t alldiff,
                    const int32_t* cons, int32_t n_cons, uint64_t* removed) {
    if (!d || !words || !removed) return CUBICS_E_INVALID;
    Model m;
    if (model_init(&m, d)) return CUBICS_E_INVALID;
    memset(removed, 0, sizeof(uint64_t) * (size_t)m.total);
    int rc = CUBICS_OK;
    int count = cons ? n_cons : d->n_cons;
    for (int i = 0; i < count && rc == CUBICS_OK; ++i) {
        int c = cons ? cons[i] : i;
        if (propagate_one(&m, c, words, removed, alldiff)) rc = CUBICS_E_OVERFLOW;
    }
    model_free(&m);
    return rc;
}
