/*
 * chroma_gen.c -- CPU generator of the BASELINE inputs for the oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see chroma_oracle.c).  It builds, on the host, the same
 * int64 CSR arrays as the product's device generators (csrc/gen.cu) and the NumPy
 * path of graph.py, from the recipe stated there:
 *   mix64 = splitmix64 finaliser of gid_rand (chroma/protocol.py:79-88);
 *   R-MAT: u = mix64((seed << 40) + e*scale + l) >> 32, src bit u >= t_ab,
 *          dst bit (t_a <= u < t_ab) || u >= t_abc, MSB first; label permutation
 *          of three (x*m_i + k_i) mod 2^bits rounds separated by x ^= x >> ceil(bits/2);
 *   random bipartite: t = ((mix64((seed << 40) + r*k + j) >> 32) * rows) >> 32;
 *   preprocess (chroma/graph.py:166-179) / preprocess_directed + to_bipartite
 *   (chroma/graph.py:182-188, 388-399): self loops and diagonal arcs dropped, both
 *   directions kept, rows sorted and de-duplicated.
 * The three implementations share no code; tests/test_generators.py compares them.
 * OpenMP parallelises the draws and the per-row sort (the result is independent of
 * the thread count: rows are sorted and de-duplicated after the parallel fill).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef uint64_t u64;
typedef uint32_t u32;

static inline u64 mix64(u64 x) {
  u64 z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct {
  u64 m[3], k[3], mask;
  int shift, on;
} perm_t;

static perm_t perm_make(u64 seed, int bits, int on) {
  perm_t p;
  for (int i = 0; i < 3; i++) {
    p.m[i] = mix64(8 * seed + 2 * (u64)i) | 1ULL;
    p.k[i] = mix64(8 * seed + 2 * (u64)i + 1);
  }
  p.mask = bits >= 64 ? ~0ULL : ((1ULL << bits) - 1);
  p.shift = (bits + 1) / 2;
  p.on = on && bits >= 1;
  return p;
}

static inline u64 perm_apply(const perm_t* p, u64 x) {
  if (!p->on) return x;
  for (int i = 0; i < 3; i++) {
    x = (x * p->m[i] + p->k[i]) & p->mask;
    if (i < 2) x ^= x >> p->shift;
  }
  return x;
}

static int cmp_i64(const void* a, const void* b) {
  const i64 x = *(const i64*)a, y = *(const i64*)b;
  return (x > y) - (x < y);
}

/* arcs (a[i], b[i]) with a[i] != b[i] (dropped arcs have a[i] < 0): symmetric,
 * sorted, de-duplicated CSR into off[n+1] / col (capacity 2*m); returns nnz */
static i64 arcs_to_csr(i64 n, i64 m, const i64* a, const i64* b, i64* off, i64* col) {
  i64* cnt = (i64*)calloc((size_t)n + 1, sizeof(i64));
  for (i64 i = 0; i < m; i++)
    if (a[i] >= 0) {
      cnt[a[i]]++;
      cnt[b[i]]++;
    }
  i64* start = (i64*)malloc(sizeof(i64) * ((size_t)n + 1));
  start[0] = 0;
  for (i64 v = 0; v < n; v++) start[v + 1] = start[v] + cnt[v];
  i64* cur = cnt;
  for (i64 v = 0; v < n; v++) cur[v] = start[v];
  for (i64 i = 0; i < m; i++)
    if (a[i] >= 0) {
      col[cur[a[i]]++] = b[i];
      col[cur[b[i]]++] = a[i];
    }
  /* sort + unique per row, in place; row lengths into cnt */
#pragma omp parallel for schedule(dynamic, 4096)
  for (i64 v = 0; v < n; v++) {
    i64* r = col + start[v];
    const i64 d = start[v + 1] - start[v];
    if (d > 1) qsort(r, (size_t)d, sizeof(i64), cmp_i64);
    i64 k = 0;
    for (i64 j = 0; j < d; j++)
      if (k == 0 || r[j] != r[k - 1]) r[k++] = r[j];
    cnt[v] = k;
  }
  off[0] = 0;
  for (i64 v = 0; v < n; v++) {
    const i64 o = off[v];
    if (o != start[v]) memmove(col + o, col + start[v], sizeof(i64) * (size_t)cnt[v]);
    off[v + 1] = o + cnt[v];
  }
  free(start);
  free(cnt);
  return off[n];
}

/* R-MAT: off[2^scale + 1], col capacity 2 * edge_factor * 2^scale */
i64 orc_gen_rmat(int scale, i64 edge_factor, u64 seed, u32 ta, u32 tab, u32 tabc, int permute, i64* off,
                 i64* col) {
  const i64 n = (i64)1 << scale, m = edge_factor << scale;
  i64* a = (i64*)malloc(sizeof(i64) * (size_t)m);
  i64* b = (i64*)malloc(sizeof(i64) * (size_t)m);
  const perm_t p = perm_make(seed, scale, permute);
#pragma omp parallel for schedule(static)
  for (i64 e = 0; e < m; e++) {
    u64 src = 0, dst = 0;
    const u64 base = (seed << 40) + (u64)e * (u64)scale;
    for (int l = 0; l < scale; l++) {
      const u32 u = (u32)(mix64(base + (u64)l) >> 32);
      src = (src << 1) | (u >= tab ? 1u : 0u);
      dst = (dst << 1) | (((u >= ta && u < tab) || u >= tabc) ? 1u : 0u);
    }
    src = perm_apply(&p, src);
    dst = perm_apply(&p, dst);
    a[e] = src == dst ? -1 : (i64)src;
    b[e] = (i64)dst;
  }
  const i64 nnz = arcs_to_csr(n, m, a, b, off, col);
  free(a);
  free(b);
  return nnz;
}

/* random bipartite (PD2): off[2*rows + 1], col capacity 2 * rows * k */
i64 orc_gen_bipartite(i64 rows, i64 k, u64 seed, i64* off, i64* col) {
  const i64 m = rows * k;
  i64* a = (i64*)malloc(sizeof(i64) * (size_t)(m > 0 ? m : 1));
  i64* b = (i64*)malloc(sizeof(i64) * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
  for (i64 e = 0; e < m; e++) {
    const i64 r = e / k;
    const i64 t = (i64)(((mix64((seed << 40) + (u64)e) >> 32) * (u64)rows) >> 32);
    a[e] = r == t ? -1 : r;
    b[e] = rows + t;
  }
  const i64 nnz = arcs_to_csr(2 * rows, m, a, b, off, col);
  free(a);
  free(b);
  return nnz;
}
