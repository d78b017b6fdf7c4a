/*
 * oracle.c -- plain, slow, obviously-correct serial CPU oracle for the BFS of arXiv 1408.1605.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header, table or helper
 * with the CUDA path (paper_1408_1605_b200/csrc); it does not know about 2D partitions, CSC
 * blocks, bitmaps, prefix sums or binary searches.  It takes a plain tuple list.
 *
 * What it computes (the definition the method reaches exactly):
 *   G = undirected simple graph with edge {s_k, d_k} for every tuple k with s_k != d_k
 *       ("We turn the graph undirected by adding, for each edge, its opposite";
 *        duplicates collapse, self-loops never matter: SPEC.md S:204).
 *   level[v]  = hop distance from root r in G, -1 if unreachable
 *               (Alg.1/Alg.2: level[r] = 0, others -1 until reached at lvl).
 *   parent[r] = r;  parent[v] = min{ u : {u,v} in E(G), level[u] = level[v]-1 }
 *               for reachable v != r (the deterministic minimum-id rule of BASELINE.json's
 *               north_star, reading R1); -1 if unreachable.
 *   m_comp    = |{ k : level[s_k] >= 0 }|, every input tuple of the traversed component,
 *               duplicates and self-loops included ("number of input edge tuples
 *               within the component traversed by the search").
 *
 * Algorithm, in the order a reader checks it:
 *   1. oracle_build: undirected adjacency by counting sort of the 2M tuple endpoints
 *      (self-loops skipped, duplicates kept -- they do not change distances or the min).
 *   2. oracle_bfs:   FIFO-queue BFS from r sets level[] (textbook BFS).
 *   3.               parent pass over the tuple list, both orientations:
 *                    if level[a] >= 0 and level[b] == level[a]+1 then parent[b] = min(parent[b], a).
 *                    Then parent[r] = r.
 *   4. oracle_mcomp: count tuples whose source is reached.
 *   5. oracle_validate: the Graph500 tree-validation invariants V1..V6.
 *   6. oracle_vstream_*: the same invariants as a streaming pass over the tuples in chunks (the
 *      caller regenerates the tuple list chunk by chunk from the seed, so full-size graphs need
 *      not be stored; SURVEY.md §8(c) "it can regenerate them from the seed"), with the tuple
 *      checks spread over the host cores (OpenMP).  Written separately from oracle_validate,
 *      which pins it (tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  uint64_t n;          /* number of vertices */
  uint64_t m;          /* number of tuples */
  const uint64_t* src; /* borrowed tuple arrays */
  const uint64_t* dst;
  uint64_t* off;       /* n+1 adjacency offsets */
  uint64_t* adj;       /* adjacency lists (undirected, self-loops skipped, duplicates kept) */
} oracle_graph;

/* Step 1: counting sort of the tuple endpoints into an undirected adjacency. Returns NULL on
 * allocation failure or an endpoint >= n. */
oracle_graph* oracle_build(uint64_t n, uint64_t m, const uint64_t* src, const uint64_t* dst) {
  oracle_graph* g = (oracle_graph*)calloc(1, sizeof(oracle_graph));
  if (!g) return NULL;
  g->n = n;
  g->m = m;
  g->src = src;
  g->dst = dst;
  g->off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  if (!g->off) { free(g); return NULL; }
  for (uint64_t k = 0; k < m; ++k) {
    uint64_t a = src[k], b = dst[k];
    if (a >= n || b >= n) { free(g->off); free(g); return NULL; }
    if (a == b) continue;
    g->off[a + 1] += 1; /* edge a -> b */
    g->off[b + 1] += 1; /* its opposite b -> a */
  }
  for (uint64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  g->adj = (uint64_t*)malloc((g->off[n] ? g->off[n] : 1) * sizeof(uint64_t));
  uint64_t* fill = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!g->adj || !fill) { free(g->adj); free(fill); free(g->off); free(g); return NULL; }
  for (uint64_t v = 0; v < n; ++v) fill[v] = g->off[v];
  for (uint64_t k = 0; k < m; ++k) {
    uint64_t a = src[k], b = dst[k];
    if (a == b) continue;
    g->adj[fill[a]++] = b;
    g->adj[fill[b]++] = a;
  }
  free(fill);
  return g;
}

void oracle_free(oracle_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->adj);
  free(g);
}

uint64_t oracle_num_adjacency(const oracle_graph* g) { return g->off[g->n]; }

/* Number of adjacency entries of v: non-self-loop tuple endpoints at v, duplicates INCLUDED (so
 * it is >= the degree of v in G, and > 0 exactly when v has a neighbour other than itself).
 * Used only as "> 0" for root eligibility (SURVEY.md §8(c) reading 14). */
uint64_t oracle_degree(const oracle_graph* g, uint64_t v) {
  return g->off[v + 1] - g->off[v];
}

/* Steps 2-3.  level[n], parent[n] are caller-allocated. Returns 0, or -2 if root >= n. */
int oracle_bfs(const oracle_graph* g, uint64_t root, int32_t* level, int64_t* parent) {
  const uint64_t n = g->n;
  if (root >= n) return -2;
  for (uint64_t v = 0; v < n; ++v) { level[v] = -1; parent[v] = -1; }
  /* 2. FIFO BFS */
  uint64_t* queue = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!queue) return -3;
  uint64_t head = 0, tail = 0;
  level[root] = 0;
  queue[tail++] = root;
  while (head < tail) {
    uint64_t u = queue[head++];
    for (uint64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      uint64_t v = g->adj[e];
      if (level[v] < 0) {
        level[v] = level[u] + 1;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  /* 3. parent = minimum neighbour one level up, from the tuple list in both orientations */
  for (uint64_t k = 0; k < g->m; ++k) {
    uint64_t a = g->src[k], b = g->dst[k];
    if (a == b) continue;
    if (level[a] >= 0 && level[b] == level[a] + 1) {
      if (parent[b] < 0 || (uint64_t)parent[b] > a) parent[b] = (int64_t)a;
    }
    if (level[b] >= 0 && level[a] == level[b] + 1) {
      if (parent[a] < 0 || (uint64_t)parent[a] > b) parent[a] = (int64_t)b;
    }
  }
  parent[root] = (int64_t)root;
  return 0;
}

/* Step 4: input tuples of the traversed component. */
uint64_t oracle_mcomp(const oracle_graph* g, const int32_t* level) {
  uint64_t c = 0;
  for (uint64_t k = 0; k < g->m; ++k)
    if (level[g->src[k]] >= 0) ++c;
  return c;
}

/* Step 5: Graph500-style validation of (level, parent) for root r against the tuple list.
 * Returns a bitmask of FAILED checks (0 = valid):
 *   bit0 V1 level[r] == 0 and parent[r] == r
 *   bit1 V2 every tree edge {parent[v], v}, v != r reached, is an input tuple (either orientation,
 *           non-self-loop)
 *   bit2 V3 level[v] == level[parent[v]] + 1 for reached v != r
 *   bit3 V4 every non-self-loop tuple with one endpoint reached has both reached, |dlevel| <= 1
 *   bit4 V5 reached set == component of r (union-find over the tuples); unreached v have
 *           level == parent == -1; reached v have parent in [0, n)
 *   bit5 V6 min rule: for every tuple (a,b), both orientations, level[a] == level[b]-1 implies
 *           parent[b] <= a
 * Streaming over the tuple list; does not need oracle_build (takes the arrays directly). */
static uint64_t uf_find(uint64_t* p, uint64_t x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}

int oracle_validate(uint64_t n, uint64_t m, const uint64_t* src, const uint64_t* dst, uint64_t root,
                    const int32_t* level, const int64_t* parent) {
  int fail = 0;
  if (root >= n) return 1;
  /* V1 */
  if (level[root] != 0 || parent[root] != (int64_t)root) fail |= 1;
  /* V5 (part): consistent unreached / range of parents */
  for (uint64_t v = 0; v < n; ++v) {
    if (level[v] < 0) {
      if (level[v] != -1 || parent[v] != -1) fail |= 16;
    } else {
      if (parent[v] < 0 || (uint64_t)parent[v] >= n) fail |= 16;
    }
  }
  if (fail & 16) return fail; /* parent[] not usable as an index */
  /* V3 */
  for (uint64_t v = 0; v < n; ++v) {
    if (v == root || level[v] < 0) continue;
    uint64_t p = (uint64_t)parent[v];
    if (level[p] < 0 || level[v] != level[p] + 1) fail |= 4;
  }
  /* V2: mark tree edges found among the tuples */
  unsigned char* found = (unsigned char*)calloc(n ? n : 1, 1);
  /* V5: union-find of the tuple graph */
  uint64_t* uf = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!found || !uf) { free(found); free(uf); return 64; }
  for (uint64_t v = 0; v < n; ++v) uf[v] = v;
  for (uint64_t k = 0; k < m; ++k) {
    uint64_t a = src[k], b = dst[k];
    if (a >= n || b >= n) { fail |= 64; continue; }
    if (a == b) continue;
    /* V2 */
    if (level[b] > 0 && (uint64_t)parent[b] == a) found[b] = 1;
    if (level[a] > 0 && (uint64_t)parent[a] == b) found[a] = 1;
    /* V4 */
    if ((level[a] >= 0) != (level[b] >= 0)) fail |= 8;
    else if (level[a] >= 0) {
      int dl = level[a] - level[b];
      if (dl > 1 || dl < -1) fail |= 8;
    }
    /* V6 */
    if (level[a] >= 0 && level[b] == level[a] + 1 && (uint64_t)parent[b] > a) fail |= 32;
    if (level[b] >= 0 && level[a] == level[b] + 1 && (uint64_t)parent[a] > b) fail |= 32;
    /* V5 union */
    uint64_t ra = uf_find(uf, a), rb = uf_find(uf, b);
    if (ra != rb) uf[ra] = rb;
  }
  for (uint64_t v = 0; v < n; ++v)
    if (v != root && level[v] > 0 && !found[v]) fail |= 2;
  uint64_t rr = uf_find(uf, root);
  for (uint64_t v = 0; v < n; ++v) {
    int in_comp = (uf_find(uf, v) == rr);
    if (in_comp != (level[v] >= 0)) fail |= 16;
  }
  free(found);
  free(uf);
  return fail;
}

/* Step 6: streaming validator.  Same bitmask as oracle_validate.
 *   begin: the per-vertex checks (V1; V5's "unreached have -1/-1, reached have a parent in
 *          [0,n)"; V3 level[v] == level[parent[v]] + 1);
 *   feed : one chunk of tuples: V2 marks the tree edges it sees, V4, V6, and the union-find of
 *          V5 (a concurrent union-find: link the larger root under the smaller one by
 *          compare-and-swap, so no cycle can form; finds halve paths with plain stores of a
 *          grand-parent, which stays an ancestor); also counts m_comp (tuples with a reached
 *          source);
 *   end  : V2 (every reached v != r had its tree edge among the tuples) and V5 (reached set ==
 *          the root's component); frees the state and returns the mask.
 * level / parent are borrowed until end. */
typedef struct {
  uint64_t n, root, mcomp;
  const int32_t* level;
  const int64_t* parent;
  unsigned char* found;
  uint64_t* uf;
  int fail;
} oracle_vstream;

oracle_vstream* oracle_vstream_begin(uint64_t n, uint64_t root, const int32_t* level, const int64_t* parent) {
  oracle_vstream* st = (oracle_vstream*)calloc(1, sizeof(oracle_vstream));
  if (!st) return NULL;
  st->n = n;
  st->root = root;
  st->level = level;
  st->parent = parent;
  if (root >= n) { st->fail = 1; return st; }
  st->found = (unsigned char*)calloc(n ? n : 1, 1);
  st->uf = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!st->found || !st->uf) { free(st->found); free(st->uf); free(st); return NULL; }
  int fail = 0;
  if (level[root] != 0 || parent[root] != (int64_t)root) fail |= 1; /* V1 */
  int64_t v;
#pragma omp parallel for reduction(| : fail) schedule(static)
  for (v = 0; v < (int64_t)n; ++v) {
    st->uf[v] = (uint64_t)v;
    if (level[v] < 0) {
      if (level[v] != -1 || parent[v] != -1) fail |= 16; /* V5: unreached are -1 / -1 */
    } else if (parent[v] < 0 || (uint64_t)parent[v] >= n) {
      fail |= 16; /* V5: a reached vertex has a parent id */
    } else if ((uint64_t)v != root) {
      const int64_t p = parent[v];
      if (level[p] < 0 || level[v] != level[p] + 1) fail |= 4; /* V3 */
    }
  }
  st->fail = fail;
  return st;
}

static uint64_t vs_find(uint64_t* uf, uint64_t x) {
  for (;;) {
    uint64_t p = __atomic_load_n(&uf[x], __ATOMIC_RELAXED);
    if (p == x) return x;
    uint64_t gp = __atomic_load_n(&uf[p], __ATOMIC_RELAXED);
    if (gp != p) __atomic_store_n(&uf[x], gp, __ATOMIC_RELAXED); /* path halving */
    x = gp;
  }
}

static void vs_union(uint64_t* uf, uint64_t a, uint64_t b) {
  for (;;) {
    uint64_t ra = vs_find(uf, a), rb = vs_find(uf, b);
    if (ra == rb) return;
    if (ra < rb) { uint64_t t = ra; ra = rb; rb = t; }
    uint64_t expect = ra; /* ra is still a root: hang it under the smaller root rb */
    if (__atomic_compare_exchange_n(&uf[ra], &expect, rb, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) return;
  }
}

void oracle_vstream_feed(oracle_vstream* st, uint64_t m, const uint64_t* src, const uint64_t* dst) {
  if (!st || (st->fail & 16) || st->root >= st->n) return; /* parent[] not usable as an index */
  const uint64_t n = st->n;
  const int32_t* level = st->level;
  const int64_t* parent = st->parent;
  int fail = 0;
  uint64_t mc = 0;
  int64_t k;
#pragma omp parallel for reduction(| : fail) reduction(+ : mc) schedule(static)
  for (k = 0; k < (int64_t)m; ++k) {
    const uint64_t a = src[k], b = dst[k];
    if (a >= n || b >= n) { fail |= 64; continue; }
    if (level[a] >= 0) ++mc; /* m_comp: tuple with a reached source, self-loops included */
    if (a == b) continue;
    /* V2: the tuple is the tree edge of b (or of a) */
    if (level[b] > 0 && (uint64_t)parent[b] == a) st->found[b] = 1;
    if (level[a] > 0 && (uint64_t)parent[a] == b) st->found[a] = 1;
    /* V4 */
    if ((level[a] >= 0) != (level[b] >= 0)) fail |= 8;
    else if (level[a] >= 0 && (level[a] - level[b] > 1 || level[b] - level[a] > 1)) fail |= 8;
    /* V6, both orientations */
    if (level[a] >= 0 && level[b] == level[a] + 1 && (uint64_t)parent[b] > a) fail |= 32;
    if (level[b] >= 0 && level[a] == level[b] + 1 && (uint64_t)parent[a] > b) fail |= 32;
    vs_union(st->uf, a, b); /* V5 */
  }
  st->fail |= fail;
  st->mcomp += mc;
}

uint64_t oracle_vstream_mcomp(const oracle_vstream* st) { return st ? st->mcomp : 0; }

int oracle_vstream_end(oracle_vstream* st) {
  if (!st) return 64;
  int fail = st->fail;
  if (!(fail & 16) && st->root < st->n) {
    const uint64_t n = st->n, root = st->root;
    const int32_t* level = st->level;
    const uint64_t rr = vs_find(st->uf, root);
    int64_t v;
#pragma omp parallel for reduction(| : fail) schedule(static)
    for (v = 0; v < (int64_t)n; ++v) {
      if ((uint64_t)v != root && level[v] > 0 && !st->found[v]) fail |= 2;   /* V2 */
      if ((vs_find(st->uf, (uint64_t)v) == rr) != (level[v] >= 0)) fail |= 16; /* V5 */
    }
  }
  free(st->found);
  free(st->uf);
  free(st);
  return fail;
}
