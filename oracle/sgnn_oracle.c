/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference update path.
 * See sgnn_oracle.h for the contract. Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj). Written in
 * plain C11 with scalar loops; compiled with -O2 -ffp-contract=off so float
 * products and sums are separately rounded exactly like the reference build.
 */
#include "sgnn_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* Errc values, src/core/error.hpp:8-19 */
enum { E_OK = 0, E_IO = 1, E_FORMAT = 2, E_DIM = 3, E_DUP = 4, E_MISSING = 5, E_UNSUPPORTED = 6,
       E_INVALID = 7, E_STALE = 8, E_CONTRACT = 9, E_NAN = 10 };

static _Thread_local char g_err[256];

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}
static void* xrealloc(void* p, size_t n) {
  p = realloc(p, n ? n : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}

/* ---- tensor.hpp:17-21 / tensor.cpp:29-58 ------------------------------ */

static float flush_zero(float x) { return x == 0.0f ? 0.0f : x; }           /* tensor.hpp:17 */
static float reduce2(int is_max, float acc, float v) {                        /* tensor.hpp:19-21 */
  return is_max ? (v > acc ? v : acc) : (v < acc ? v : acc);
}
static void ewise_reduce_into(int is_max, const float* v, float* acc, uint32_t d) { /* tensor.cpp:29-32 */
  for (uint32_t i = 0; i < d; ++i) acc[i] = reduce2(is_max, acc[i], v[i]);
}
/* tensor.cpp:41-53: ascending column order, bias after the dot product, -0 flushed */
static void matvec_affine(const float* w, uint32_t rows, uint32_t cols, const float* x, const float* bias,
                          float* out) {
  for (uint32_t r = 0; r < rows; ++r) {
    const float* row = w + (size_t)r * cols;
    float acc = 0.0f;
    for (uint32_t c = 0; c < cols; ++c) acc += row[c] * x[c];
    if (bias) acc += bias[r];
    out[r] = flush_zero(acc);
  }
}
static void relu_inplace(float* x, uint32_t d) {                              /* tensor.cpp:55-58 */
  for (uint32_t i = 0; i < d; ++i) x[i] = x[i] > 0.0f ? x[i] : 0.0f;
}
static int rows_equal(const float* a, const float* b, uint32_t d) {           /* engine.cpp:135-138 */
  return memcmp(a, b, (size_t)d * sizeof(float)) == 0;
}

void orc_matvec_affine(const float* w, uint32_t rows, uint32_t cols, const float* x, const float* bias,
                       float* out) {
  matvec_affine(w, rows, cols, x, bias, out);
}

/* ---- dynamic arrays ---------------------------------------------------- */

typedef struct { uint32_t* a; uint32_t n, cap; } u32vec;

static void u32_reserve(u32vec* v, uint32_t cap) {
  if (cap <= v->cap) return;
  uint32_t nc = v->cap ? v->cap : 4;
  while (nc < cap) nc *= 2;
  v->a = (uint32_t*)xrealloc(v->a, (size_t)nc * sizeof(uint32_t));
  v->cap = nc;
}
static void u32_push(u32vec* v, uint32_t x) {
  u32_reserve(v, v->n + 1);
  v->a[v->n++] = x;
}
static uint32_t lower_bound(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
static void u32_insert_at(u32vec* v, uint32_t pos, uint32_t x) {
  u32_reserve(v, v->n + 1);
  memmove(v->a + pos + 1, v->a + pos, (size_t)(v->n - pos) * sizeof(uint32_t));
  v->a[pos] = x;
  v->n++;
}
static void u32_erase_at(u32vec* v, uint32_t pos) {
  memmove(v->a + pos, v->a + pos + 1, (size_t)(v->n - pos - 1) * sizeof(uint32_t));
  v->n--;
}

/* ---- u64 -> payload open-addressing map (std::map / unordered_map stand-in) */

typedef struct { uint64_t* keys; int64_t* vals; size_t cap, n; } u64map;  /* key 0 = empty; keys stored +1 */

static void map_init(u64map* m, size_t want) {
  size_t cap = 16;
  while (cap < 2 * want + 2) cap *= 2;
  m->keys = (uint64_t*)xcalloc(cap, sizeof(uint64_t));
  m->vals = (int64_t*)xcalloc(cap, sizeof(int64_t));
  m->cap = cap;
  m->n = 0;
}
static void map_free(u64map* m) { free(m->keys); free(m->vals); memset(m, 0, sizeof *m); }
static size_t map_slot(const u64map* m, uint64_t key) {
  uint64_t k = key + 1, h = k * 0x9E3779B97F4A7C15ull;
  size_t i = (size_t)(h >> 17) & (m->cap - 1);
  while (m->keys[i] && m->keys[i] != k) i = (i + 1) & (m->cap - 1);
  return i;
}
static int64_t* map_find(const u64map* m, uint64_t key) {
  size_t i = map_slot(m, key);
  return m->keys[i] ? &m->vals[i] : NULL;
}
static void map_put(u64map* m, uint64_t key, int64_t val);
static void map_grow(u64map* m) {
  u64map nm;
  map_init(&nm, m->cap);
  for (size_t i = 0; i < m->cap; ++i)
    if (m->keys[i]) map_put(&nm, m->keys[i] - 1, m->vals[i]);
  map_free(m);
  *m = nm;
}
static void map_put(u64map* m, uint64_t key, int64_t val) {
  if (2 * (m->n + 1) > m->cap) map_grow(m);
  size_t i = map_slot(m, key);
  if (!m->keys[i]) { m->keys[i] = key + 1; m->n++; }
  m->vals[i] = val;
}
static void map_clear(u64map* m) {
  memset(m->keys, 0, m->cap * sizeof(uint64_t));
  m->n = 0;
}

/* ---- DynamicGraph, graph.hpp:27-56 / graph.cpp:10-131 ------------------- */

enum { OP_INSERT = 0, OP_DELETE = 1 };
typedef struct { int op; uint32_t src, dst; } delta_t;

typedef struct {
  uint32_t n;
  uint64_t m;
  u32vec* out;
  u32vec* in;
  delta_t* pending;
  size_t npending, cap_pending;
  int prev_valid;
} graph_t;

static int graph_init(graph_t* g, uint32_t n) {                              /* graph.cpp:10-13 */
  memset(g, 0, sizeof *g);
  if (n == 0) { snprintf(g_err, sizeof g_err, "graph must have at least one node"); return E_INVALID; }
  g->n = n;
  g->out = (u32vec*)xcalloc(n, sizeof(u32vec));
  g->in = (u32vec*)xcalloc(n, sizeof(u32vec));
  g->prev_valid = 1;
  return E_OK;
}
static void graph_free(graph_t* g) {
  for (uint32_t i = 0; i < g->n; ++i) { free(g->out[i].a); free(g->in[i].a); }
  free(g->out); free(g->in); free(g->pending);
}
static int has_edge(const graph_t* g, uint32_t s, uint32_t d) {              /* graph.cpp:20-25 */
  const u32vec* o = &g->out[s];
  uint32_t p = lower_bound(o->a, o->n, d);
  return p < o->n && o->a[p] == d;
}
static void insert_adj(graph_t* g, uint32_t s, uint32_t d) {                  /* graph.cpp:27-33 */
  u32vec* o = &g->out[s];
  u32_insert_at(o, lower_bound(o->a, o->n, d), d);
  u32vec* i = &g->in[d];
  u32_insert_at(i, lower_bound(i->a, i->n, s), s);
  g->m++;
}
static void erase_adj(graph_t* g, uint32_t s, uint32_t d) {                   /* graph.cpp:35-41 */
  u32vec* o = &g->out[s];
  u32_erase_at(o, lower_bound(o->a, o->n, d));
  u32vec* i = &g->in[d];
  u32_erase_at(i, lower_bound(i->a, i->n, s));
  g->m--;
}
static int add_edge(graph_t* g, uint32_t s, uint32_t d) {                     /* graph.cpp:43-50 */
  if (g->npending) { snprintf(g_err, sizeof g_err, "add_edge is only valid with no pending delta"); return E_INVALID; }
  if (s >= g->n || d >= g->n) {
    snprintf(g_err, sizeof g_err, "node id out of range: %u", s >= g->n ? s : d);
    return E_INVALID;
  }
  if (has_edge(g, s, d)) { snprintf(g_err, sizeof g_err, "duplicate edge %u->%u", s, d); return E_DUP; }
  insert_adj(g, s, d);
  return E_OK;
}
static uint64_t edge_key(uint32_t s, uint32_t d) { return ((uint64_t)s << 32) | d; }

/* graph.cpp:52-79: validate the whole batch against an overlay, then mutate. */
static int apply_delta(graph_t* g, const delta_t* delta, size_t cnt) {
  u64map overlay;
  map_init(&overlay, cnt);
  for (size_t i = 0; i < cnt; ++i) {
    const delta_t* d = &delta[i];
    if (d->src >= g->n || d->dst >= g->n) {
      snprintf(g_err, sizeof g_err, "node id out of range: %u", d->src >= g->n ? d->src : d->dst);
      map_free(&overlay);
      return E_INVALID;
    }
    uint64_t key = edge_key(d->src, d->dst);
    int64_t* it = map_find(&overlay, key);
    int present = it ? (int)*it : has_edge(g, d->src, d->dst);
    if (d->op == OP_INSERT && present) {
      snprintf(g_err, sizeof g_err, "insert of existing edge %u->%u", d->src, d->dst);
      map_free(&overlay);
      return E_DUP;
    }
    if (d->op == OP_DELETE && !present) {
      snprintf(g_err, sizeof g_err, "delete of missing edge %u->%u", d->src, d->dst);
      map_free(&overlay);
      return E_MISSING;
    }
    map_put(&overlay, key, d->op == OP_INSERT);
  }
  map_free(&overlay);
  for (size_t i = 0; i < cnt; ++i) {
    if (delta[i].op == OP_INSERT) insert_adj(g, delta[i].src, delta[i].dst);
    else erase_adj(g, delta[i].src, delta[i].dst);
    if (g->npending == g->cap_pending) {
      g->cap_pending = g->cap_pending ? 2 * g->cap_pending : 64;
      g->pending = (delta_t*)xrealloc(g->pending, g->cap_pending * sizeof(delta_t));
    }
    g->pending[g->npending++] = delta[i];
  }
  g->prev_valid = 1;
  return E_OK;
}

/* graph.cpp:87-106: previous-timestamp neighbourhood = current list with the
 * pending delta inverted in reverse order. dir 0 = out, 1 = in. */
static void neighbors_prev(const graph_t* g, uint32_t u, int dir, u32vec* res) {
  const u32vec* cur = dir == 0 ? &g->out[u] : &g->in[u];
  res->n = 0;
  u32_reserve(res, cur->n + 1);
  memcpy(res->a, cur->a, (size_t)cur->n * sizeof(uint32_t));
  res->n = cur->n;
  for (size_t k = g->npending; k-- > 0;) {
    const delta_t* d = &g->pending[k];
    uint32_t self = dir == 0 ? d->src : d->dst;
    if (self != u) continue;
    uint32_t other = dir == 0 ? d->dst : d->src;
    uint32_t pos = lower_bound(res->a, res->n, other);
    if (d->op == OP_INSERT) {
      if (pos < res->n && res->a[pos] == other) u32_erase_at(res, pos);
    } else {
      if (pos == res->n || res->a[pos] != other) u32_insert_at(res, pos, other);
    }
  }
}

typedef struct { uint64_t key; size_t seq; int op; } keyed_t;
static int cmp_keyed(const void* a, const void* b) {
  const keyed_t* x = (const keyed_t*)a;
  const keyed_t* y = (const keyed_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* graph.cpp:113-131: net effect per (src,dst), sorted by key. */
static size_t net_edge_delta(const delta_t* delta, size_t cnt, delta_t** out) {
  keyed_t* k = (keyed_t*)xmalloc(cnt * sizeof(keyed_t));
  for (size_t i = 0; i < cnt; ++i) {
    k[i].key = edge_key(delta[i].src, delta[i].dst);
    k[i].seq = i;
    k[i].op = delta[i].op;
  }
  qsort(k, cnt, sizeof(keyed_t), cmp_keyed);
  delta_t* net = (delta_t*)xmalloc(cnt * sizeof(delta_t));
  size_t nn = 0;
  for (size_t i = 0; i < cnt;) {
    size_t j = i;
    while (j + 1 < cnt && k[j + 1].key == k[i].key) ++j;
    int initial = !(k[i].op == OP_INSERT);   /* Presence{!present, present} of the first op */
    int final = k[j].op == OP_INSERT;
    if (initial != final) {
      net[nn].op = final ? OP_INSERT : OP_DELETE;
      net[nn].src = (uint32_t)(k[i].key >> 32);
      net[nn].dst = (uint32_t)(k[i].key & 0xffffffffu);
      nn++;
    }
    i = j + 1;
  }
  free(k);
  *out = net;
  return nn;
}

/* ---- model (model.cpp:184-218 dims, 238-284 run_combination/run_prefix) */

typedef struct {
  orc_op* ops;
  int nops;
  int is_max;
  int k;
  int* part_begin;
  int* part_end;
  int* part_agg;
  uint32_t* stage_dims;  /* [0] = message dim of layer 1 .. [k] = output dim */
  int has_prefix, has_user;
  int* user_ops_in_part;  /* number of user_apply ops after the aggregate of each partition */
} model_t;

static int model_init(model_t* m, const orc_op* ops, int nops, int is_max, uint32_t input_dim) {
  memset(m, 0, sizeof *m);
  m->ops = (orc_op*)xmalloc((size_t)nops * sizeof(orc_op));
  memcpy(m->ops, ops, (size_t)nops * sizeof(orc_op));
  m->nops = nops;
  m->is_max = is_max;
  int* aggs = (int*)xmalloc((size_t)(nops + 1) * sizeof(int));
  int na = 0;
  for (int i = 0; i < nops; ++i)
    if (ops[i].kind == ORC_OP_AGGREGATE) aggs[na++] = i;
  if (na == 0) { free(aggs); snprintf(g_err, sizeof g_err, "model has no aggregation line"); return E_FORMAT; }
  m->k = na;
  m->part_begin = (int*)xmalloc((size_t)na * sizeof(int));
  m->part_end = (int*)xmalloc((size_t)na * sizeof(int));
  m->part_agg = (int*)xmalloc((size_t)na * sizeof(int));
  m->user_ops_in_part = (int*)xcalloc((size_t)na, sizeof(int));
  for (int p = 0; p < na; ++p) {                                      /* model.cpp:87-95 */
    m->part_begin[p] = p == 0 ? 0 : aggs[p];
    m->part_end[p] = p + 1 < na ? aggs[p + 1] : nops;
    m->part_agg[p] = aggs[p];
  }
  free(aggs);
  m->has_prefix = m->part_agg[0] > 0;
  m->stage_dims = (uint32_t*)xmalloc((size_t)(na + 1) * sizeof(uint32_t));
  uint32_t d = input_dim;
  int nd = 0;
  for (int p = 0; p < na; ++p) {
    for (int i = m->part_begin[p]; i < m->part_end[p]; ++i) {
      const orc_op* op = &ops[i];
      if (op->kind == ORC_OP_AGGREGATE) {
        m->stage_dims[nd++] = d;
      } else if (op->kind == ORC_OP_LINEAR) {
        if (op->cols != d) { snprintf(g_err, sizeof g_err, "weight expects input length %u, got %u", op->cols, d); return E_DIM; }
        d = op->rows;
      } else if (op->kind == ORC_OP_SAGE_SELF) {
        if (op->cols != m->stage_dims[p] || op->rows != d) { snprintf(g_err, sizeof g_err, "sage_self dims"); return E_DIM; }
        m->has_user = 1;
        if (i > m->part_agg[p]) m->user_ops_in_part[p]++;
      } else if (op->kind == ORC_OP_GIN_SELF) {
        if (d != m->stage_dims[p]) { snprintf(g_err, sizeof g_err, "gin_self dims"); return E_DIM; }
        m->has_user = 1;
        if (i > m->part_agg[p]) m->user_ops_in_part[p]++;
      }
    }
  }
  m->stage_dims[nd] = d;
  return E_OK;
}
static void model_free(model_t* m) {
  free(m->ops); free(m->part_begin); free(m->part_end); free(m->part_agg); free(m->stage_dims);
  free(m->user_ops_in_part);
}
static uint32_t message_dim(const model_t* m, int layer) { return m->stage_dims[layer - 1]; }
static uint32_t max_dim(const model_t* m) {
  uint32_t d = 0;
  for (int i = 0; i <= m->k; ++i) if (m->stage_dims[i] > d) d = m->stage_dims[i];
  for (int i = 0; i < m->nops; ++i)
    if (m->ops[i].kind == ORC_OP_LINEAR && m->ops[i].rows > d) d = m->ops[i].rows;
  return d;
}

/* Self-message provider (ApplyContext, model.hpp:100-104). */
typedef const float* (*self_fn)(void* ctx);

/* model.cpp:238-269 + hooks.cpp:24-36. x holds alpha (length message_dim(p+1))
 * on entry; the result (length message_dim(p+2)) is written to out. */
static void run_combination(const model_t* m, int p, const float* alpha, float* out, self_fn self, void* ctx,
                            float* t0, float* t1) {
  uint32_t d = message_dim(m, p + 1);
  float* x = t0;
  float* y = t1;
  memcpy(x, alpha, (size_t)d * sizeof(float));
  for (int i = m->part_agg[p] + 1; i < m->part_end[p]; ++i) {
    const orc_op* op = &m->ops[i];
    switch (op->kind) {
      case ORC_OP_LINEAR:
        matvec_affine(op->w, op->rows, op->cols, x, op->bias, y);
        d = op->rows;
        { float* t = x; x = y; y = t; }
        break;
      case ORC_OP_RELU:
        relu_inplace(x, d);
        break;
      case ORC_OP_SAGE_SELF: {                                         /* hooks.cpp:24-29 */
        const float* sm = self(ctx);
        matvec_affine(op->w, op->rows, op->cols, sm, NULL, y);
        for (uint32_t j = 0; j < d; ++j) x[j] = flush_zero(x[j] + y[j]);
        break;
      }
      case ORC_OP_GIN_SELF: {                                          /* hooks.cpp:31-36 */
        const float* sm = self(ctx);
        const float scale = 1.0f + op->eps;
        for (uint32_t j = 0; j < d; ++j) x[j] = flush_zero(x[j] + scale * sm[j]);
        break;
      }
      default:
        break;
    }
  }
  memcpy(out, x, (size_t)d * sizeof(float));
}

/* model.cpp:271-284 */
static void run_prefix(const model_t* m, const float* feat, uint32_t F, float* out, float* t0, float* t1) {
  uint32_t d = F;
  float* x = t0;
  float* y = t1;
  memcpy(x, feat, (size_t)d * sizeof(float));
  for (int i = 0; i < m->part_agg[0]; ++i) {
    const orc_op* op = &m->ops[i];
    if (op->kind == ORC_OP_LINEAR) {
      matvec_affine(op->w, op->rows, op->cols, x, op->bias, y);
      d = op->rows;
      float* t = x; x = y; y = t;
    } else if (op->kind == ORC_OP_RELU) {
      relu_inplace(x, d);
    }
  }
  memcpy(out, x, (size_t)d * sizeof(float));
}

/* ---- CheckpointStore, checkpoint.hpp:25-61 / checkpoint.cpp:11-82 ------- */

enum { ST_MSG = 0, ST_AGG = 1 };

typedef struct {
  uint32_t n;
  int k;
  uint32_t* msg_dim;   /* [l-1], l = 1..k+1 */
  float** msg;
  float** agg;         /* [l-1], l = 1..k, dim = msg_dim[l-1] */
  u64map undo;         /* key -> index into undo_rows */
  float** undo_rows;
  size_t n_undo, cap_undo;
  uint64_t l1_msg_rows, other_rows;   /* FetchCounters, checkpoint.hpp:15-19 */
} store_t;

static void store_init(store_t* s, const model_t* m, uint32_t n) {
  memset(s, 0, sizeof *s);
  s->n = n;
  s->k = m->k;
  s->msg_dim = (uint32_t*)xmalloc((size_t)(m->k + 1) * sizeof(uint32_t));
  s->msg = (float**)xmalloc((size_t)(m->k + 1) * sizeof(float*));
  s->agg = (float**)xmalloc((size_t)m->k * sizeof(float*));
  for (int l = 1; l <= m->k + 1; ++l) {
    s->msg_dim[l - 1] = message_dim(m, l);
    s->msg[l - 1] = (float*)xcalloc((size_t)n * s->msg_dim[l - 1], sizeof(float));
  }
  for (int l = 1; l <= m->k; ++l) s->agg[l - 1] = (float*)xcalloc((size_t)n * s->msg_dim[l - 1], sizeof(float));
  map_init(&s->undo, 64);
}
static void store_free(store_t* s) {
  for (int l = 0; l <= s->k; ++l) free(s->msg[l]);
  for (int l = 0; l < s->k; ++l) free(s->agg[l]);
  for (size_t i = 0; i < s->n_undo; ++i) free(s->undo_rows[i]);
  free(s->undo_rows); free(s->msg); free(s->agg); free(s->msg_dim);
  map_free(&s->undo);
}
static uint32_t store_dim(const store_t* s, int layer) { return s->msg_dim[layer - 1]; }
static float* table_row(const store_t* s, int layer, int stage, uint32_t v) {
  uint32_t d = store_dim(s, layer);
  float* t = stage == ST_MSG ? s->msg[layer - 1] : s->agg[layer - 1];
  return t + (size_t)v * d;
}
static uint64_t store_key(int layer, uint32_t v, int stage) {                  /* checkpoint.cpp:40-43 */
  return ((uint64_t)(stage == ST_AGG) << 63) | ((uint64_t)layer << 32) | v;
}
static void count_read(store_t* s, int layer, int stage) {                     /* checkpoint.cpp:45-50 */
  if (layer == 1 && stage == ST_MSG) s->l1_msg_rows++; else s->other_rows++;
}
static const float* read_prev(store_t* s, int layer, uint32_t v, int stage) {  /* checkpoint.cpp:52-57 */
  count_read(s, layer, stage);
  int64_t* it = map_find(&s->undo, store_key(layer, v, stage));
  if (it) return s->undo_rows[*it];
  return table_row(s, layer, stage, v);
}
static const float* read_current(store_t* s, int layer, uint32_t v, int stage) { /* checkpoint.cpp:59-62 */
  count_read(s, layer, stage);
  return table_row(s, layer, stage, v);
}
static void write_current(store_t* s, int layer, uint32_t v, int stage, const float* x) { /* 64-76 */
  uint32_t d = store_dim(s, layer);
  float* row = table_row(s, layer, stage, v);
  uint64_t key = store_key(layer, v, stage);
  if (!map_find(&s->undo, key)) {
    if (s->n_undo == s->cap_undo) {
      s->cap_undo = s->cap_undo ? 2 * s->cap_undo : 64;
      s->undo_rows = (float**)xrealloc(s->undo_rows, s->cap_undo * sizeof(float*));
    }
    float* copy = (float*)xmalloc((size_t)d * sizeof(float));
    memcpy(copy, row, (size_t)d * sizeof(float));
    s->undo_rows[s->n_undo] = copy;
    map_put(&s->undo, key, (int64_t)s->n_undo);
    s->n_undo++;
  }
  memcpy(row, x, (size_t)d * sizeof(float));
}
static void commit_round(store_t* s) {                                         /* checkpoint.cpp:78-82 */
  for (size_t i = 0; i < s->n_undo; ++i) free(s->undo_rows[i]);
  s->n_undo = 0;
  map_clear(&s->undo);
}

/* ---- engine (engine.hpp / engine.cpp) ---------------------------------- */

typedef struct { int op; uint32_t target; uint32_t msg_idx; } event_t;  /* engine.hpp:13-20, op 0 Add 1 Del */

typedef struct {
  event_t* ev;
  size_t nev, cap_ev;
  float* msgs;
  size_t nmsg, cap_msg;
  uint32_t d;
} queue_t;

static uint32_t q_push_message(queue_t* q, const float* v) {                  /* engine.cpp:7-10 */
  if (q->nmsg == q->cap_msg) {
    q->cap_msg = q->cap_msg ? 2 * q->cap_msg : 64;
    q->msgs = (float*)xrealloc(q->msgs, q->cap_msg * q->d * sizeof(float));
  }
  memcpy(q->msgs + q->nmsg * q->d, v, (size_t)q->d * sizeof(float));
  return (uint32_t)q->nmsg++;
}
static void q_push_event(queue_t* q, int op, uint32_t target, uint32_t idx) {  /* engine.cpp:12-15 */
  if (q->nev == q->cap_ev) {
    q->cap_ev = q->cap_ev ? 2 * q->cap_ev : 64;
    q->ev = (event_t*)xrealloc(q->ev, q->cap_ev * sizeof(event_t));
  }
  q->ev[q->nev].op = op;
  q->ev[q->nev].target = target;
  q->ev[q->nev].msg_idx = idx;
  q->nev++;
}

typedef struct { uint32_t target; float* payload; } user_event_t;
typedef struct { user_event_t* a; size_t n, cap; } user_queue_t;

struct orc_engine {
  graph_t g;
  model_t model;
  float* features;
  uint32_t F;
  store_t store;
  int dup_seed, baseline;
  int emit_changed_only; /* north-star item 5: no next-layer events from unchanged messages (not in the reference) */
  queue_t* queues;
  user_queue_t* uqueues;
  u32vec* dirty;
  uint64_t* last;   /* k * ORC_NUM_COUNTERS + 7 */
};

/* Self message for the engine: user-event stash or a counted read_current
 * (engine.cpp:118-133). */
typedef struct { store_t* s; int layer; uint32_t v; const float* stashed; } engine_ctx;
static const float* engine_self(void* c) {
  engine_ctx* x = (engine_ctx*)c;
  if (x->stashed) return x->stashed;
  return read_current(x->s, x->layer, x->v, ST_MSG);
}
/* Uncounted table access (checkpoint.cpp:88-99 TableApplyContext). */
typedef struct { const float* row; } table_ctx;
static const float* table_self(void* c) { return ((table_ctx*)c)->row; }

/* classify, engine.cpp:45-78. kinds: 0 NoDeletion 1 DeletionNoEffect 2 Covered 3 Exposed */
int orc_classify(const float* alpha_prev, const float* del, const float* add, uint32_t dim, int is_max) {
  if (!del) return 0;
  int any_reset = 0, covered = 1;
  for (uint32_t i = 0; i < dim; ++i) {
    if (alpha_prev[i] == del[i]) {
      any_reset = 1;
      if (!add || reduce2(is_max, del[i], add[i]) != add[i]) covered = 0;
    }
  }
  if (!any_reset) return 1;
  if (add && covered) return 2;
  return 3;
}

/* checkpoint.cpp:105-145 */
static void init_full_inference(orc_engine* e) {
  const model_t* m = &e->model;
  store_t* s = &e->store;
  uint32_t md = max_dim(m);
  if (md < e->F) md = e->F;
  float* t0 = (float*)xmalloc(md * sizeof(float));
  float* t1 = (float*)xmalloc(md * sizeof(float));
  float* a = (float*)xmalloc(md * sizeof(float));
  float* nx = (float*)xmalloc(md * sizeof(float));
  for (uint32_t v = 0; v < e->g.n; ++v) {
    const float* f = e->features + (size_t)v * e->F;
    if (m->has_prefix) {
      run_prefix(m, f, e->F, nx, t0, t1);
      write_current(s, 1, v, ST_MSG, nx);
    } else {
      write_current(s, 1, v, ST_MSG, f);
    }
  }
  for (int l = 1; l <= m->k; ++l) {
    uint32_t d = store_dim(s, l);
    for (uint32_t v = 0; v < e->g.n; ++v) {
      const u32vec* nb = &e->g.in[v];
      memset(a, 0, d * sizeof(float));
      if (nb->n) {
        memcpy(a, table_row(s, l, ST_MSG, nb->a[0]), d * sizeof(float));
        for (uint32_t i = 1; i < nb->n; ++i) ewise_reduce_into(m->is_max, table_row(s, l, ST_MSG, nb->a[i]), a, d);
      }
      write_current(s, l, v, ST_AGG, a);
      table_ctx ctx = {table_row(s, l, ST_MSG, v)};
      run_combination(m, l - 1, a, nx, table_self, &ctx, t0, t1);
      write_current(s, l + 1, v, ST_MSG, nx);
    }
  }
  commit_round(s);
  s->l1_msg_rows = s->other_rows = 0;
  free(t0); free(t1); free(a); free(nx);
}

orc_engine* orc_create(uint32_t num_nodes, const uint32_t* src, const uint32_t* dst, uint64_t num_edges,
                       const float* features, uint32_t feature_len, const orc_op* ops, int num_ops, int is_max,
                       int* status) {
  orc_engine* e = (orc_engine*)xcalloc(1, sizeof(orc_engine));
  int st = graph_init(&e->g, num_nodes);
  if (st) { free(e); *status = st; return NULL; }
  for (uint64_t i = 0; i < num_edges; ++i) {
    st = add_edge(&e->g, src[i], dst[i]);
    if (st) { graph_free(&e->g); free(e); *status = st; return NULL; }
  }
  st = model_init(&e->model, ops, num_ops, is_max, feature_len);
  if (st) { graph_free(&e->g); free(e); *status = st; return NULL; }
  e->F = feature_len;
  e->features = (float*)xmalloc((size_t)num_nodes * feature_len * sizeof(float));
  for (size_t i = 0; i < (size_t)num_nodes * feature_len; ++i) {
    if (features[i] != features[i]) {
      snprintf(g_err, sizeof g_err, "NaN in features");
      orc_destroy(e);
      *status = E_NAN;
      return NULL;
    }
    e->features[i] = flush_zero(features[i]);
  }
  store_init(&e->store, &e->model, num_nodes);
  int k = e->model.k;
  e->queues = (queue_t*)xcalloc((size_t)k, sizeof(queue_t));
  for (int l = 1; l <= k; ++l) e->queues[l - 1].d = message_dim(&e->model, l);
  e->uqueues = (user_queue_t*)xcalloc((size_t)k, sizeof(user_queue_t));
  e->dirty = (u32vec*)xcalloc((size_t)k, sizeof(u32vec));
  e->last = (uint64_t*)xcalloc((size_t)k * ORC_NUM_COUNTERS + 7, sizeof(uint64_t));
  init_full_inference(e);
  *status = E_OK;
  return e;
}

void orc_destroy(orc_engine* e) {
  if (!e) return;
  int k = e->model.k;
  if (e->queues) {
    for (int l = 0; l < k; ++l) { free(e->queues[l].ev); free(e->queues[l].msgs); }
    for (int l = 0; l < k; ++l) {
      for (size_t i = 0; i < e->uqueues[l].n; ++i) free(e->uqueues[l].a[i].payload);
      free(e->uqueues[l].a);
      free(e->dirty[l].a);
    }
    free(e->queues); free(e->uqueues); free(e->dirty);
    store_free(&e->store);
  }
  free(e->last);
  free(e->features);
  model_free(&e->model);
  graph_free(&e->g);
  free(e);
}

int orc_set_option(orc_engine* e, const char* name, int64_t value) {    /* capi.cpp:280-292 */
  if (!strcmp(name, "baseline_counters")) e->baseline = value != 0;
  else if (!strcmp(name, "duplicate_seed_events")) e->dup_seed = value != 0;
  else if (!strcmp(name, "emit_changed_only")) e->emit_changed_only = value != 0;
  else { snprintf(g_err, sizeof g_err, "unknown option: %s", name); return E_INVALID; }
  return E_OK;
}
int orc_num_layers(const orc_engine* e) { return e->model.k; }
const char* orc_last_error(void) { return g_err; }
uint64_t orc_num_edges(const orc_engine* e) { return e->g.m; }

/* ---- baseline counters, baseline.cpp:101-232 --------------------------- */

/* affected_area (baseline.cpp:101-131): returns |area(hops)| and fills
 * members (unsorted) of the final area. */
static size_t affected_area(const graph_t* g, const delta_t* net, size_t nnet, int hops, u32vec* members) {
  char* reached = (char*)xcalloc(g->n, 1);
  u32vec frontier = {0}, next = {0};
  members->n = 0;
  for (size_t i = 0; i < nnet; ++i) {
    uint32_t us[2] = {net[i].src, net[i].dst};
    for (int j = 0; j < 2; ++j)
      if (!reached[us[j]]) { reached[us[j]] = 1; u32_push(&frontier, us[j]); u32_push(members, us[j]); }
  }
  for (int l = 0; l < hops; ++l) {
    next.n = 0;
    for (uint32_t i = 0; i < frontier.n; ++i) {
      const u32vec* o = &g->out[frontier.a[i]];
      for (uint32_t j = 0; j < o->n; ++j)
        if (!reached[o->a[j]]) { reached[o->a[j]] = 1; u32_push(&next, o->a[j]); }
    }
    for (uint32_t i = 0; i < next.n; ++i) u32_push(members, next.a[i]);
    u32vec t = frontier; frontier = next; next = t;
  }
  free(reached); free(frontier.a); free(next.a);
  return members->n;
}

/* affected_fetch_count (baseline.cpp:149-173 need sets, 209-222 count) */
static uint64_t affected_fetch_count(const graph_t* g, const delta_t* net, size_t nnet, const model_t* m) {
  u32vec need = {0};
  affected_area(g, net, nnet, m->k, &need);      /* need[k+1] = area(k) */
  uint64_t count = 0;
  uint64_t* per_level_sum = (uint64_t*)xcalloc((size_t)m->k + 2, sizeof(uint64_t));
  /* need[l] for l = k..1: need[l+1] plus the in-neighbourhood of need[l+1] */
  u32vec cur = need;  /* need[l+1] */
  char* in_set = (char*)xmalloc(g->n);
  for (int l = m->k; l >= 1; --l) {
    /* count for layer l uses need[l+1] = cur */
    uint64_t self = m->user_ops_in_part[l - 1] > 0 ? 1 : 0;
    for (uint32_t i = 0; i < cur.n; ++i) count += g->in[cur.a[i]].n + self;
    memset(in_set, 0, g->n);
    u32vec nxt = {0};
    for (uint32_t i = 0; i < cur.n; ++i) {
      uint32_t v = cur.a[i];
      if (!in_set[v]) { in_set[v] = 1; u32_push(&nxt, v); }
      const u32vec* in = &g->in[v];
      for (uint32_t j = 0; j < in->n; ++j)
        if (!in_set[in->a[j]]) { in_set[in->a[j]] = 1; u32_push(&nxt, in->a[j]); }
    }
    free(cur.a);
    cur = nxt;   /* need[l] */
  }
  if (m->has_prefix) count += cur.n;   /* |need[1]| */
  free(cur.a);
  free(in_set);
  free(per_level_sum);
  return count;
}

/* baseline.cpp:224-232 */
static uint64_t full_fetch_count(const graph_t* g, const model_t* m) {
  uint64_t count = m->has_prefix ? g->n : 0;
  for (int l = 1; l <= m->k; ++l) {
    uint64_t self = m->user_ops_in_part[l - 1] > 0 ? 1 : 0;
    for (uint32_t v = 0; v < g->n; ++v) count += g->in[v].n + self;
  }
  return count;
}

/* ---- group_and_reduce, engine.cpp:27-43 -------------------------------- */

typedef struct { uint32_t target; size_t idx; } tgt_idx;
static int cmp_tgt(const void* a, const void* b) {
  const tgt_idx* x = (const tgt_idx*)a;
  const tgt_idx* y = (const tgt_idx*)b;
  if (x->target != y->target) return x->target < y->target ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

typedef struct {
  uint32_t target;
  int has_del, has_add;
  float* del;
  float* add;
} group_t;

static size_t group_and_reduce(const queue_t* q, int is_max, group_t** out, float** arena) {
  tgt_idx* order = (tgt_idx*)xmalloc(q->nev * sizeof(tgt_idx));
  for (size_t i = 0; i < q->nev; ++i) { order[i].target = q->ev[i].target; order[i].idx = i; }
  qsort(order, q->nev, sizeof(tgt_idx), cmp_tgt);
  size_t ng = 0;
  for (size_t i = 0; i < q->nev; ++i)
    if (i == 0 || order[i].target != order[i - 1].target) ng++;
  group_t* g = (group_t*)xcalloc(ng, sizeof(group_t));
  float* mem = (float*)xmalloc(2 * ng * q->d * sizeof(float) + sizeof(float));
  size_t gi = (size_t)-1;
  for (size_t i = 0; i < q->nev; ++i) {
    if (i == 0 || order[i].target != order[i - 1].target) {
      gi++;
      g[gi].target = order[i].target;
      g[gi].del = mem + 2 * gi * q->d;
      g[gi].add = g[gi].del + q->d;
    }
    const event_t* ev = &q->ev[order[i].idx];
    const float* msg = q->msgs + (size_t)ev->msg_idx * q->d;
    int* has = ev->op == 1 ? &g[gi].has_del : &g[gi].has_add;
    float* slot = ev->op == 1 ? g[gi].del : g[gi].add;
    if (!*has) { memcpy(slot, msg, q->d * sizeof(float)); *has = 1; }
    else ewise_reduce_into(is_max, msg, slot, q->d);
  }
  free(order);
  *out = g;
  *arena = mem;
  return ng;
}

typedef struct { uint32_t target; size_t idx; } stash_ent;
static int cmp_stash(const void* a, const void* b) {
  const stash_ent* x = (const stash_ent*)a;
  const stash_ent* y = (const stash_ent*)b;
  if (x->target != y->target) return x->target < y->target ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* ---- Engine::process_update_round, engine.cpp:171-319 ------------------ */

int orc_apply(orc_engine* e, const char* opc, const uint32_t* src, const uint32_t* dst, size_t count) {
  const int k = e->model.k;
  const int is_max = e->model.is_max;
  store_t* s = &e->store;
  graph_t* g = &e->g;
  delta_t* delta = (delta_t*)xmalloc((count + 1) * sizeof(delta_t));
  for (size_t i = 0; i < count; ++i) {                                 /* capi.cpp:269-273 */
    if (opc[i] != '+' && opc[i] != '-') {
      free(delta);
      snprintf(g_err, sizeof g_err, "op must be '+' or '-'");
      return E_INVALID;
    }
    delta[i].op = opc[i] == '+' ? OP_INSERT : OP_DELETE;
    delta[i].src = src[i];
    delta[i].dst = dst[i];
  }
  for (int l = 0; l < k; ++l) e->dirty[l].n = 0;                      /* 174-177 */
  s->l1_msg_rows = s->other_rows = 0;

  int st = apply_delta(g, delta, count);                                /* 179 */
  if (st) { free(delta); return st; }
  delta_t* net = NULL;
  size_t nnet = net_edge_delta(g->pending, g->npending, &net);          /* 180 */

  uint64_t* stats = (uint64_t*)xcalloc((size_t)k * ORC_NUM_COUNTERS + 7, sizeof(uint64_t));
  uint32_t md = max_dim(&e->model);
  float* t0 = (float*)xmalloc(md * sizeof(float));
  float* t1 = (float*)xmalloc(md * sizeof(float));
  float* alpha_new = (float*)xmalloc(md * sizeof(float));
  float* m_next = (float*)xmalloc(md * sizeof(float));
  float* m_prev = (float*)xmalloc(md * sizeof(float));
  u32vec nb = {0};

  for (int l = 1; l <= k; ++l) {
    uint64_t* ls = stats + (size_t)(l - 1) * ORC_NUM_COUNTERS;
    const uint64_t before = s->l1_msg_rows + s->other_rows;
    queue_t* q = &e->queues[l - 1];
    const uint32_t d = q->d;

    for (size_t i = 0; i < nnet; ++i) {                                 /* seed_edge_events, 101-112 */
      const float* m = net[i].op == OP_DELETE ? read_prev(s, l, net[i].src, ST_MSG)
                                              : read_current(s, l, net[i].src, ST_MSG);
      q_push_event(q, net[i].op == OP_DELETE ? 1 : 0, net[i].dst, q_push_message(q, m));
    }
    if (e->dup_seed) {                                                  /* 192-195 */
      size_t n0 = q->nev;
      for (size_t i = 0; i < n0; ++i) q_push_event(q, q->ev[i].op, q->ev[i].target, q->ev[i].msg_idx);
    }

    group_t* groups = NULL;
    float* garena = NULL;
    size_t ng = group_and_reduce(q, is_max, &groups, &garena);          /* 197 */

    /* stash: std::map<NodeId, Vec>, later entries overwrite (201-203) */
    user_queue_t* uq = &e->uqueues[l - 1];
    stash_ent* stash = (stash_ent*)xmalloc((uq->n + 1) * sizeof(stash_ent));
    for (size_t i = 0; i < uq->n; ++i) { stash[i].target = uq->a[i].target; stash[i].idx = i; }
    qsort(stash, uq->n, sizeof(stash_ent), cmp_stash);
    size_t ns = 0;
    for (size_t i = 0; i < uq->n; ++i) {   /* keep the last payload per target */
      if (ns && stash[ns - 1].target == stash[i].target) stash[ns - 1] = stash[i];
      else stash[ns++] = stash[i];
    }

    ls[ORC_EVENTS] = q->nev;
    ls[ORC_TARGETS] = ng;
    ls[ORC_USER_TARGETS] = ns;

    size_t gi = 0, si = 0;
    while (gi < ng || si < ns) {                                        /* 212-292 */
      const group_t* grp = NULL;
      const float* self_new = NULL;
      uint32_t v;
      if (gi < ng && (si == ns || groups[gi].target <= stash[si].target)) {
        grp = &groups[gi];
        v = grp->target;
        if (si < ns && stash[si].target == v) { self_new = uq->a[stash[si].idx].payload; ++si; }
        ++gi;
      } else {
        v = stash[si].target;
        self_new = uq->a[stash[si].idx].payload;
        ++si;
      }

      int alpha_changed = 0;
      if (grp) {
        const float* alpha_prev = read_prev(s, l, v, ST_AGG);           /* 233 */
        neighbors_prev(g, v, 1, &nb);
        if (!grp->has_del && nb.n == 0) {                               /* 234-238 */
          memcpy(alpha_new, grp->add, d * sizeof(float));
          ls[ORC_NO_DEL]++;
        } else {
          int kind = orc_classify(alpha_prev, grp->has_del ? grp->del : NULL, grp->has_add ? grp->add : NULL, d,
                                  is_max);
          ls[ORC_NO_DEL + kind]++;
          if (kind == 3) {                                              /* recompute, 89-99 */
            const u32vec* in = &g->in[v];
            memset(alpha_new, 0, d * sizeof(float));
            if (in->n) {
              memcpy(alpha_new, read_current(s, l, in->a[0], ST_MSG), d * sizeof(float));
              for (uint32_t i = 1; i < in->n; ++i)
                ewise_reduce_into(is_max, read_current(s, l, in->a[i], ST_MSG), alpha_new, d);
            }
            ls[ORC_RECOMPUTES]++;
          } else {                                                      /* incremental, 80-87 */
            memcpy(alpha_new, alpha_prev, d * sizeof(float));
            if (grp->has_add) ewise_reduce_into(is_max, grp->add, alpha_new, d);
          }
        }
        alpha_changed = !rows_equal(alpha_new, alpha_prev, d);          /* 253 */
      }

      if (!alpha_changed && !self_new) continue;                        /* 258 */

      if (alpha_changed) {
        write_current(s, l, v, ST_AGG, alpha_new);
      } else if (!grp) {
        memcpy(alpha_new, read_current(s, l, v, ST_AGG), d * sizeof(float));
      }
      u32_push(&e->dirty[l - 1], v);

      engine_ctx ctx = {s, l, v, self_new};
      run_combination(&e->model, l - 1, alpha_new, m_next, engine_self, &ctx, t0, t1);
      const uint32_t dn = message_dim(&e->model, l + 1);

      if (l < k) {                                                      /* 271-289 */
        memcpy(m_prev, read_prev(s, l + 1, v, ST_MSG), dn * sizeof(float));
        const int msg_changed = !rows_equal(m_next, m_prev, dn);
        write_current(s, l + 1, v, ST_MSG, m_next);
        queue_t* nq = &e->queues[l];
        /* emit_changed_only: a source whose m_{l+1} is bitwise unchanged sends
           Del(m) + Add(m) pairs that can change no aggregate (the reference
           sends them, engine.cpp:276-283); skip them. Tables and dirty sets are
           unchanged; events / targets / conditions / fetch counters shrink. */
        if (e->emit_changed_only && !msg_changed) continue;
        uint32_t idx_old = q_push_message(nq, m_prev);
        uint32_t idx_new = q_push_message(nq, m_next);
        neighbors_prev(g, v, 0, &nb);
        for (uint32_t i = 0; i < nb.n; ++i) q_push_event(nq, 1, nb.a[i], idx_old);
        const u32vec* out = &g->out[v];
        for (uint32_t i = 0; i < out->n; ++i) q_push_event(nq, 0, out->a[i], idx_new);
        if (e->model.has_user && msg_changed) {
          user_queue_t* nu = &e->uqueues[l];
          if (nu->n == nu->cap) {
            nu->cap = nu->cap ? 2 * nu->cap : 64;
            nu->a = (user_event_t*)xrealloc(nu->a, nu->cap * sizeof(user_event_t));
          }
          nu->a[nu->n].target = v;
          nu->a[nu->n].payload = (float*)xmalloc(dn * sizeof(float));
          memcpy(nu->a[nu->n].payload, m_next, dn * sizeof(float));
          nu->n++;
        }
      } else {
        write_current(s, k + 1, v, ST_MSG, m_next);
      }
    }

    for (size_t i = 0; i < uq->n; ++i) free(uq->a[i].payload);
    uq->n = 0;
    free(stash);
    free(groups);
    free(garena);
    q->nev = 0;                                                         /* 294 */
    q->nmsg = 0;
    ls[ORC_DIRTY] = e->dirty[l - 1].n;
    ls[ORC_FETCH_ROWS] = s->l1_msg_rows + s->other_rows - before;
  }

  uint64_t* tail = stats + (size_t)k * ORC_NUM_COUNTERS;
  tail[0] = count;
  if (e->model.has_prefix) {                                            /* 300-307 */
    tail[2] = 0;
    tail[1] = s->l1_msg_rows + s->other_rows;
  } else {
    tail[2] = s->l1_msg_rows;
    tail[1] = s->other_rows;
  }
  if (e->baseline) {                                                    /* 309-314 */
    tail[3] = 1;
    tail[4] = affected_fetch_count(g, net, nnet, &e->model);
    tail[5] = full_fetch_count(g, &e->model);
    u32vec area = {0};
    tail[6] = affected_area(g, net, nnet, k, &area);
    free(area.a);
  }
  g->npending = 0;                                                      /* graph_.commit(), graph.cpp:108-111 */
  g->prev_valid = 0;
  commit_round(s);

  memcpy(e->last, stats, ((size_t)k * ORC_NUM_COUNTERS + 7) * sizeof(uint64_t));
  free(stats); free(t0); free(t1); free(alpha_new); free(m_next); free(m_prev); free(nb.a);
  free(net); free(delta);
  return E_OK;
}

void orc_last_stats(const orc_engine* e, uint64_t* out) {
  memcpy(out, e->last, ((size_t)e->model.k * ORC_NUM_COUNTERS + 7) * sizeof(uint64_t));
}

uint32_t orc_dim(const orc_engine* e, int layer, int stage) {
  if (layer < 1 || layer > e->model.k + 1 || (stage == ST_AGG && layer > e->model.k)) return 0;
  return store_dim(&e->store, layer);
}

void orc_table(const orc_engine* e, int layer, int stage, float* out) {
  uint32_t d = store_dim(&e->store, layer);
  const float* t = stage == ST_MSG ? e->store.msg[layer - 1] : e->store.agg[layer - 1];
  memcpy(out, t, (size_t)e->store.n * d * sizeof(float));
}

uint64_t orc_dirty(const orc_engine* e, int layer, uint32_t* buf, uint64_t cap) {
  const u32vec* v = &e->dirty[layer - 1];
  if (buf) memcpy(buf, v->a, (size_t)(cap < v->n ? cap : v->n) * sizeof(uint32_t));
  return v->n;
}

/* baseline::full_inference (baseline.cpp:67-99) + verify_against_full (234-256) */
int orc_verify(const orc_engine* e, uint32_t* out_layer, uint32_t* out_stage, uint32_t* out_node,
               uint32_t* out_index) {
  const model_t* m = &e->model;
  const int k = m->k;
  const uint32_t n = e->g.n;
  float** msg = (float**)xmalloc((size_t)(k + 1) * sizeof(float*));
  float** agg = (float**)xmalloc((size_t)k * sizeof(float*));
  for (int l = 1; l <= k + 1; ++l) msg[l - 1] = (float*)xcalloc((size_t)n * message_dim(m, l), sizeof(float));
  for (int l = 1; l <= k; ++l) agg[l - 1] = (float*)xcalloc((size_t)n * message_dim(m, l), sizeof(float));
  uint32_t md = max_dim(m);
  if (md < e->F) md = e->F;
  float* t0 = (float*)xmalloc(md * sizeof(float));
  float* t1 = (float*)xmalloc(md * sizeof(float));
  for (uint32_t v = 0; v < n; ++v) {
    const float* f = e->features + (size_t)v * e->F;
    if (m->has_prefix) run_prefix(m, f, e->F, msg[0] + (size_t)v * message_dim(m, 1), t0, t1);
    else memcpy(msg[0] + (size_t)v * e->F, f, e->F * sizeof(float));
  }
  for (int l = 1; l <= k; ++l) {
    uint32_t d = message_dim(m, l), dn = message_dim(m, l + 1);
    for (uint32_t v = 0; v < n; ++v) {
      float* a = agg[l - 1] + (size_t)v * d;
      const u32vec* nb = &e->g.in[v];
      if (nb->n) {
        memcpy(a, msg[l - 1] + (size_t)nb->a[0] * d, d * sizeof(float));
        for (uint32_t i = 1; i < nb->n; ++i) ewise_reduce_into(m->is_max, msg[l - 1] + (size_t)nb->a[i] * d, a, d);
      }
      table_ctx ctx = {msg[l - 1] + (size_t)v * d};
      run_combination(m, l - 1, a, msg[l] + (size_t)v * dn, table_self, &ctx, t0, t1);
    }
  }
  int rc = 0;
  for (int l = 1; l <= k + 1 && !rc; ++l) {
    for (int st = 0; st < (l <= k ? 2 : 1) && !rc; ++st) {
      uint32_t d = message_dim(m, l);
      const float* got = st == 0 ? e->store.msg[l - 1] : e->store.agg[l - 1];
      const float* want = st == 0 ? msg[l - 1] : agg[l - 1];
      for (uint32_t v = 0; v < n && !rc; ++v)
        for (uint32_t i = 0; i < d; ++i)
          if (memcmp(&got[(size_t)v * d + i], &want[(size_t)v * d + i], sizeof(float)) != 0) {
            if (out_layer) *out_layer = (uint32_t)l;
            if (out_stage) *out_stage = (uint32_t)st;
            if (out_node) *out_node = v;
            if (out_index) *out_index = i;
            rc = 11;
            break;
          }
    }
  }
  for (int l = 0; l <= k; ++l) free(msg[l]);
  for (int l = 0; l < k; ++l) free(agg[l]);
  free(msg); free(agg); free(t0); free(t1);
  return rc;
}
