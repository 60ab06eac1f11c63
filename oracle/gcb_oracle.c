/*
 * gcb_oracle.c -- CPU restatement of the reference TOCAB hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_1904_02241_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * never links or calls it.
 *
 * Every routine restates one reference function (file:line into
 * /root/reference/pkg/src/gcb) with the same floating-point operation order, so
 * outputs are bit-identical to the reference (pinned by tests/golden and the
 * sha256 checksums in SURVEY.md section 8c).  Compile with -ffp-contract=off: the
 * reference's numba loops emit separate vmulsd/vaddsd (no FMA).
 *
 * Conventions: int64_t sizes; vertex ids uint32_t (graph.py:4-6); CSR row offsets
 * int64_t; edge weights double.  Functions return 0 on success, nonzero on bad
 * arguments / allocation failure.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------------------
 * PCG64 (numpy's default bit generator, XSL-RR 128/64).  Used by
 * _generate_rmat graph.py:371-386 via np.random.default_rng(seed).random(m).
 * random(): state = state*M + inc; u = xsl_rr(state); double = (u >> 11) * 2^-53.
 * The (state, inc) pair after seeding is taken from numpy (PCG64(seed).state).
 * ------------------------------------------------------------------------- */
static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static inline uint64_t pcg_output(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

/* affine map (mult, plus) equal to `delta` LCG steps */
static void pcg_jump(u128 delta, u128 inc, u128 *mult, u128 *plus) {
  u128 acc_m = 1, acc_p = 0, cur_m = PCG_MULT, cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  *mult = acc_m;
  *plus = acc_p;
}

static inline double pcg_next_double(u128 *s, u128 inc) {
  *s = *s * PCG_MULT + inc;
  return (double)(pcg_output(*s) >> 11) * (1.0 / 9007199254740992.0);
}

/* First `count` doubles of the stream (for pinning against numpy). */
int orc_pcg64_doubles(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                      uint64_t inc_lo, int64_t skip, int64_t count, double *out) {
  u128 s = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  u128 jm, jp;
  pcg_jump((u128)skip, inc, &jm, &jp);
  s = jm * s + jp;
  for (int64_t i = 0; i < count; ++i) out[i] = pcg_next_double(&s, inc);
  return 0;
}

/* R-MAT endpoints, graph.py:371-386.  Level l (MSB first) of edge i uses draw
 * l*m + i.  src_bit = r >= a+b; dst_bit = (a <= r < a+b) | (r >= a+b+c).
 * Outputs uint32 ids (scale <= 31 so ids fit). */
int orc_rmat_edges(int scale, int64_t m, uint64_t st_hi, uint64_t st_lo,
                   uint64_t inc_hi, uint64_t inc_lo, double a, double t_ab,
                   double t_abc, uint32_t *src, uint32_t *dst, int threads) {
  if (scale < 1 || scale > 31 || m < 0) return 1;
  u128 s0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  memset(src, 0, (size_t)m * sizeof(uint32_t));
  memset(dst, 0, (size_t)m * sizeof(uint32_t));
  int nt = threads > 0 ? threads : 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
  {
    int tid = 0, T = 1;
#ifdef _OPENMP
    tid = omp_get_thread_num();
    T = omp_get_num_threads();
#endif
    int64_t chunk = (m + T - 1) / T;
    int64_t i0 = (int64_t)tid * chunk, i1 = i0 + chunk;
    if (i1 > m) i1 = m;
    if (i0 < i1) {
      for (int l = 0; l < scale; ++l) {
        u128 jm, jp;
        pcg_jump((u128)((u128)l * (u128)m + (u128)i0), inc, &jm, &jp);
        u128 s = jm * s0 + jp;
        for (int64_t i = i0; i < i1; ++i) {
          double r = pcg_next_double(&s, inc);
          uint32_t sb = r >= t_ab;
          uint32_t db = ((r >= a) && (r < t_ab)) || (r >= t_abc);
          src[i] = (src[i] << 1) | sb;
          dst[i] = (dst[i] << 1) | db;
        }
      }
    }
  }
  (void)nt;
  return 0;
}

/* ---------------------------------------------------------------------------
 * from_edges graph.py:110-130: np.lexsort((dst, src)) (stable), row counts by
 * bincount(src), col = dst[order], weights = w[order].  Restated as two stable
 * LSD counting sorts (by dst, then by src), which yields the same permutation.
 * ------------------------------------------------------------------------- */
static int counting_pass(int64_t n, int64_t m, const uint32_t *key,
                         const int64_t *in, int64_t *out, int64_t *cnt) {
  memset(cnt, 0, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) cnt[key[in ? in[i] : i] + 1]++;
  for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
  for (int64_t i = 0; i < m; ++i) {
    int64_t e = in ? in[i] : i;
    out[cnt[key[e]]++] = e;
  }
  return 0;
}

int orc_from_edges(int64_t n, int64_t m, const uint32_t *src, const uint32_t *dst,
                   const double *w, int64_t *row_offsets, uint32_t *col,
                   double *w_out) {
  for (int64_t i = 0; i < m; ++i)
    if ((int64_t)src[i] >= n || (int64_t)dst[i] >= n) return 1;
  int64_t *o1 = (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t));
  int64_t *o2 = (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t));
  int64_t *cnt = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
  if (!o1 || !o2 || !cnt) { free(o1); free(o2); free(cnt); return 2; }
  counting_pass(n, m, dst, NULL, o1, cnt);
  counting_pass(n, m, src, o1, o2, cnt);
  memset(row_offsets, 0, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) row_offsets[src[i] + 1]++;
  for (int64_t v = 0; v < n; ++v) row_offsets[v + 1] += row_offsets[v];
  for (int64_t i = 0; i < m; ++i) {
    col[i] = dst[o2[i]];
    if (w && w_out) w_out[i] = w[o2[i]];
  }
  free(o1); free(o2); free(cnt);
  return 0;
}

/* transpose graph.py:133-138 == from_edges(col, edge_sources) */
int orc_transpose(int64_t n, int64_t m, const int64_t *ro, const uint32_t *col,
                  const double *w, int64_t *ro_t, uint32_t *col_t, double *w_t) {
  uint32_t *srcs = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  if (!srcs) return 2;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) srcs[e] = (uint32_t)v;
  int rc = orc_from_edges(n, m, col, srcs, w, ro_t, col_t, w_t);
  free(srcs);
  return rc;
}

/* ---------------------------------------------------------------------------
 * partition_tocab blocking.py:189-253.  Stable partition of edges by col//W;
 * each (block,row) run becomes a local row; id_map ascending per block;
 * lro_arena holds per-block (n_local+1)-long local offset segments.
 * ------------------------------------------------------------------------- */
int orc_partition_sizes(int64_t n, int64_t m, const int64_t *ro, const uint32_t *col,
                        int64_t width, int64_t *num_blocks, int64_t *total_rows) {
  if (width < 1 || ro[n] != m) return 1;
  int64_t B = (n + width - 1) / width, L = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t prev = -1;
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      int64_t b = col[e] / width;
      if (b != prev) { L++; prev = b; }
    }
  }
  *num_blocks = B;
  *total_rows = L;
  return 0;
}

int orc_partition_fill(int64_t n, int64_t m, const int64_t *ro, const uint32_t *col,
                       const double *w, int64_t width, int64_t B,
                       int64_t *row_starts, int64_t *lro_arena, uint32_t *id_map,
                       int64_t *edge_starts, uint32_t *col_arena, double *w_arena) {
  if (ro[n] != m) return 1;
  int64_t *epos = (int64_t *)calloc((size_t)(B + 1), sizeof(int64_t));
  int64_t *rpos = (int64_t *)calloc((size_t)(B + 1), sizeof(int64_t));
  if (!epos || !rpos) { free(epos); free(rpos); return 2; }
  memset(edge_starts, 0, (size_t)(B + 1) * sizeof(int64_t));
  memset(row_starts, 0, (size_t)(B + 1) * sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) {
    int64_t prev = -1;
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      int64_t b = col[e] / width;
      edge_starts[b + 1]++;
      if (b != prev) { row_starts[b + 1]++; prev = b; }
    }
  }
  for (int64_t b = 0; b < B; ++b) {
    edge_starts[b + 1] += edge_starts[b];
    row_starts[b + 1] += row_starts[b];
  }
  for (int64_t b = 0; b < B; ++b) {
    epos[b] = edge_starts[b];
    rpos[b] = row_starts[b];
    lro_arena[row_starts[b] + b] = 0; /* first local offset of every segment */
  }
  /* rows ascending; inside a row cols ascending => stable by block */
  for (int64_t v = 0; v < n; ++v) {
    int64_t prev = -1;
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      int64_t b = col[e] / width;
      if (b != prev) {
        id_map[rpos[b]] = (uint32_t)v;
        rpos[b]++;
        prev = b;
      }
      int64_t p = epos[b]++;
      col_arena[p] = col[e];
      if (w && w_arena) w_arena[p] = w[e];
      /* local offset of the row end == edges placed so far in block b */
      lro_arena[rpos[b] - 1 + b + 1] = epos[b] - edge_starts[b];
    }
  }
  free(epos); free(rpos);
  return 0;
}

/* BlockedGraph.range_bounds blocking.py:151-173 (searchsorted side=left). */
int orc_range_bounds(int64_t n, int64_t B, const int64_t *row_starts,
                     const uint32_t *id_map, int64_t k, int64_t *bounds) {
  if (k < 1) return 1;
  int64_t R = n ? (n + k - 1) / k : 0;
  for (int64_t b = 0; b < B; ++b) {
    int64_t rs = row_starts[b], re = row_starts[b + 1];
    int64_t *row = bounds + b * (R + 1);
    row[0] = rs;
    int64_t p = rs;
    for (int64_t j = 1; j <= R; ++j) {
      int64_t lim = j * k;
      while (p < re && (int64_t)id_map[p] < lim) ++p;
      row[j] = p;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * _gather_rows kernels.py:155-161 / _gather_rows_weighted 164-170:
 * sequential f64 sum in storage order (weighted: separate mul, then add).
 * ------------------------------------------------------------------------- */
int orc_gather_rows(const double *values, const double *weights,
                    const uint32_t *col, const int64_t *offsets, int64_t lo,
                    int64_t hi, double *out, int threads) {
  (void)threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4096) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t r = lo; r < hi; ++r) {
    double s = 0.0;
    if (weights) {
      for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) {
        double p = weights[e] * values[col[e]];
        s += p;
      }
    } else {
      for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) s += values[col[e]];
    }
    out[r] = s;
  }
  return 0;
}

/* compute_contributions kernels.py:185-191 (IEEE division; dangling -> 0). */
static void contributions(int64_t n, const double *ranks, const int64_t *deg,
                          double *out, int threads) {
  (void)threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t v = 0; v < n; ++v) out[v] = deg[v] > 0 ? ranks[v] / (double)deg[v] : 0.0;
}

/* numpy's pairwise summation (umath loops: pairwise_sum, PW_BLOCKSIZE 128,
 * 8 accumulators) over |a-b|, so `delta` equals float(np.abs(new-old).sum()). */
static double pairwise_absdiff(const double *a, const double *b, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += fabs(a[i] - b[i]);
    return res;
  } else if (n <= 128) {
    double r[8], res;
    for (int j = 0; j < 8; ++j) r[j] = fabs(a[j] - b[j]);
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += fabs(a[i + j] - b[i + j]);
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += fabs(a[i] - b[i]);
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_absdiff(a, b, n2) + pairwise_absdiff(a + n2, b + n2, n - n2);
  }
}

double orc_pairwise_absdiff(const double *a, const double *b, int64_t n) {
  return pairwise_absdiff(a, b, n);
}

/* accumulate_ranges kernels.py:300-321: per vertex, block-ordered adds from 0. */
static void merge_blocks(int64_t n, int64_t B, const int64_t *row_starts,
                         const uint32_t *id_map, const double *partials, double *sums) {
  memset(sums, 0, (size_t)n * sizeof(double));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t i = row_starts[b]; i < row_starts[b + 1]; ++i)
      sums[id_map[i]] += partials[i];
}

int orc_accumulate(int64_t n, int64_t B, const int64_t *row_starts,
                   const uint32_t *id_map, const double *partials, double *sums) {
  merge_blocks(n, B, row_starts, id_map, partials, sums);
  return 0;
}

/* per-block pull partials (kernels.py:333-347) */
static void pull_partials(int64_t B, const int64_t *row_starts, const int64_t *lro,
                          const int64_t *edge_starts, const uint32_t *col,
                          const double *w, const double *values, double *partials,
                          int threads) {
  for (int64_t b = 0; b < B; ++b) {
    int64_t rs = row_starts[b], re = row_starts[b + 1], es = edge_starts[b];
    const int64_t *off = lro + rs + b;
    (void)threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4096) num_threads(threads > 0 ? threads : 1)
#endif
    for (int64_t i = 0; i < re - rs; ++i) {
      double s = 0.0;
      if (w) {
        for (int64_t e = off[i]; e < off[i + 1]; ++e) {
          double p = w[es + e] * values[col[es + e]];
          s += p;
        }
      } else {
        for (int64_t e = off[i]; e < off[i + 1]; ++e) s += values[col[es + e]];
      }
      partials[rs + i] = s;
    }
  }
}

/* push-direction sums (process_block_push kernels.py:285-297): per block the
 * bincount walks storage order, i.e. rows (sources) ascending. */
static void push_sums(int64_t n, int64_t B, const int64_t *row_starts,
                      const int64_t *lro, const uint32_t *id_map,
                      const int64_t *edge_starts, const uint32_t *col,
                      const double *w, const double *values, double *sums) {
  memset(sums, 0, (size_t)n * sizeof(double));
  for (int64_t b = 0; b < B; ++b) {
    int64_t rs = row_starts[b], re = row_starts[b + 1], es = edge_starts[b];
    const int64_t *off = lro + rs + b;
    for (int64_t i = 0; i < re - rs; ++i) {
      double c = values[id_map[rs + i]];
      for (int64_t e = off[i]; e < off[i + 1]; ++e) {
        double p = w ? w[es + e] * c : c;
        sums[col[es + e]] += p;
      }
    }
  }
}

/* pr_blocked kernels.py:367-405 over a tocab blocking (pull or push).
 * direction: 0 pull, 1 push.  deg = _blocked_out_degrees kernels.py:324-330. */
int orc_pr_blocked(int direction, int64_t n, int64_t m, int64_t B,
                   const int64_t *row_starts, const int64_t *lro,
                   const uint32_t *id_map, const int64_t *edge_starts,
                   const uint32_t *col, double damping, double tol, int max_iters,
                   double *ranks, int *iterations, int *converged, int threads) {
  int64_t L = row_starts[B];
  int64_t *deg = (int64_t *)calloc((size_t)(n ? n : 1), sizeof(int64_t));
  double *c = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *sums = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *nr = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *partials = (double *)malloc((size_t)(L ? L : 1) * sizeof(double));
  if (!deg || !c || !sums || !nr || !partials) {
    free(deg); free(c); free(sums); free(nr); free(partials);
    return 2;
  }
  if (direction == 0) {
    for (int64_t e = 0; e < m; ++e) deg[col[e]]++;
  } else {
    for (int64_t b = 0; b < B; ++b)
      for (int64_t i = row_starts[b]; i < row_starts[b + 1]; ++i) {
        const int64_t *off = lro + row_starts[b] + b;
        int64_t li = i - row_starts[b];
        deg[id_map[i]] += off[li + 1] - off[li];
      }
  }
  for (int64_t v = 0; v < n; ++v) ranks[v] = 1.0 / (double)n;
  double base = (1.0 - damping) / (double)n;
  int it = 0, conv = 0;
  for (int k = 0; k < max_iters; ++k) {
    contributions(n, ranks, deg, c, threads);
    if (direction == 0) {
      pull_partials(B, row_starts, lro, edge_starts, col, NULL, c, partials, threads);
      merge_blocks(n, B, row_starts, id_map, partials, sums);
    } else {
      push_sums(n, B, row_starts, lro, id_map, edge_starts, col, NULL, c, sums);
    }
    for (int64_t v = 0; v < n; ++v) {
      double t = damping * sums[v];
      nr[v] = base + t;
    }
    double delta = pairwise_absdiff(nr, ranks, n);
    memcpy(ranks, nr, (size_t)n * sizeof(double));
    ++it;
    if (delta < tol) { conv = 1; break; }
  }
  *iterations = it;
  *converged = conv;
  free(deg); free(c); free(sums); free(nr); free(partials);
  return 0;
}

/* pr_baseline kernels.py:207-268 (deterministic): pull over the transpose with
 * deg = bincount(col); push over the forward graph with deg = out-degree. */
int orc_pr_baseline(int direction, int64_t n, int64_t m, const int64_t *ro,
                    const uint32_t *col, const int64_t *deg_in, double damping,
                    double tol, int max_iters, double *ranks, int *iterations,
                    int *converged, int threads) {
  int64_t *deg = (int64_t *)calloc((size_t)(n ? n : 1), sizeof(int64_t));
  double *c = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *sums = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *nr = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  if (!deg || !c || !sums || !nr) { free(deg); free(c); free(sums); free(nr); return 2; }
  if (deg_in) memcpy(deg, deg_in, (size_t)n * sizeof(int64_t));
  else if (direction == 0) for (int64_t e = 0; e < m; ++e) deg[col[e]]++;
  else for (int64_t v = 0; v < n; ++v) deg[v] = ro[v + 1] - ro[v];
  for (int64_t v = 0; v < n; ++v) ranks[v] = 1.0 / (double)n;
  double base = (1.0 - damping) / (double)n;
  int it = 0, conv = 0;
  for (int k = 0; k < max_iters; ++k) {
    contributions(n, ranks, deg, c, threads);
    if (direction == 0) {
      orc_gather_rows(c, NULL, col, ro, 0, n, sums, threads);
    } else {
      memset(sums, 0, (size_t)n * sizeof(double));
      for (int64_t v = 0; v < n; ++v)
        for (int64_t e = ro[v]; e < ro[v + 1]; ++e) sums[col[e]] += c[v];
    }
    for (int64_t v = 0; v < n; ++v) {
      double t = damping * sums[v];
      nr[v] = base + t;
    }
    double delta = pairwise_absdiff(nr, ranks, n);
    memcpy(ranks, nr, (size_t)n * sizeof(double));
    ++it;
    if (delta < tol) { conv = 1; break; }
  }
  *iterations = it;
  *converged = conv;
  free(deg); free(c); free(sums); free(nr);
  return 0;
}

/* spmv_blocked kernels.py:431-487 (tocab pull / push). */
int orc_spmv_blocked(int direction, int64_t n, int64_t B, const int64_t *row_starts,
                     const int64_t *lro, const uint32_t *id_map,
                     const int64_t *edge_starts, const uint32_t *col, const double *w,
                     const double *x, double *y, int threads) {
  if (direction == 0) {
    int64_t L = row_starts[B];
    double *partials = (double *)malloc((size_t)(L ? L : 1) * sizeof(double));
    if (!partials) return 2;
    pull_partials(B, row_starts, lro, edge_starts, col, w, x, partials, threads);
    merge_blocks(n, B, row_starts, id_map, partials, y);
    free(partials);
  } else {
    push_sums(n, B, row_starts, lro, id_map, edge_starts, col, w, x, y);
  }
  return 0;
}

/* spmv kernels.py:412-428 over a plain CSR. */
int orc_spmv(int direction, int64_t n, const int64_t *ro, const uint32_t *col,
             const double *w, const double *x, double *y, int threads) {
  if (direction == 0) return orc_gather_rows(x, w, col, ro, 0, n, y, threads);
  memset(y, 0, (size_t)n * sizeof(double));
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      double p = w ? x[v] * w[e] : x[v];
      y[col[e]] += p;
    }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Traversal.  BFS depth (traversal.py:179-209): level-synchronous, INF = 2^31-1.
 * Direction choice does not change depths (test_acceptance c6), so the oracle
 * is a plain queue BFS.  Returns the number of non-empty levels.
 * ------------------------------------------------------------------------- */
int orc_bfs(int64_t n, const int64_t *ro, const uint32_t *col, int64_t source,
            int32_t *depth, int64_t *num_levels) {
  if (source < 0 || source >= n) return 1;
  for (int64_t v = 0; v < n; ++v) depth[v] = INT32_MAX;
  uint32_t *q = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  if (!q) return 2;
  int64_t head = 0, tail = 0;
  q[tail++] = (uint32_t)source;
  depth[source] = 0;
  int32_t maxd = 0;
  while (head < tail) {
    uint32_t u = q[head++];
    for (int64_t e = ro[u]; e < ro[u + 1]; ++e) {
      uint32_t v = col[e];
      if (depth[v] == INT32_MAX) {
        depth[v] = depth[u] + 1;
        if (depth[v] > maxd) maxd = depth[v];
        q[tail++] = v;
      }
    }
  }
  *num_levels = (int64_t)maxd + 1;
  free(q);
  return 0;
}

/* SSSP with non-negative integer weights (no reference code):
 * binary-heap Dijkstra; parallel edges act as their minimum weight.
 * dist = INT64_MAX when unreachable. */
typedef struct { int64_t d; uint32_t v; } heap_item;

static void heap_push(heap_item *h, int64_t *sz, heap_item it) {
  int64_t i = (*sz)++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h[p].d < it.d || (h[p].d == it.d && h[p].v <= it.v)) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = it;
}

static heap_item heap_pop(heap_item *h, int64_t *sz) {
  heap_item top = h[0], last = h[--(*sz)];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    heap_item best = last;
    if (l < *sz && (h[l].d < best.d || (h[l].d == best.d && h[l].v < best.v))) { s = l; best = h[l]; }
    if (r < *sz && (h[r].d < best.d || (h[r].d == best.d && h[r].v < best.v))) { s = r; best = h[r]; }
    if (s == i) break;
    h[i] = h[s];
    i = s;
  }
  if (*sz > 0) h[i] = last;
  return top;
}

int orc_sssp(int64_t n, int64_t m, const int64_t *ro, const uint32_t *col,
             const int64_t *w, int64_t source, int64_t *dist) {
  if (source < 0 || source >= n) return 1;
  for (int64_t v = 0; v < n; ++v) dist[v] = INT64_MAX;
  heap_item *h = (heap_item *)malloc((size_t)(m + 1) * sizeof(heap_item));
  if (!h) return 2;
  int64_t sz = 0;
  dist[source] = 0;
  heap_item s0 = {0, (uint32_t)source};
  heap_push(h, &sz, s0);
  while (sz > 0) {
    heap_item it = heap_pop(h, &sz);
    if (it.d != dist[it.v]) continue;
    for (int64_t e = ro[it.v]; e < ro[it.v + 1]; ++e) {
      if (w[e] < 0) { free(h); return 1; }
      int64_t nd = it.d + w[e];
      uint32_t v = col[e];
      if (nd < dist[v]) {
        dist[v] = nd;
        heap_item ni = {nd, v};
        heap_push(h, &sz, ni);
      }
    }
  }
  free(h);
  return 0;
}

/* Weakly connected components, canonical label = minimum vertex id
 * (no reference code).  Union-find with union by min id. */
static uint32_t uf_find(uint32_t *p, uint32_t x) {
  while (p[x] != x) {
    p[x] = p[p[x]];
    x = p[x];
  }
  return x;
}

int orc_cc(int64_t n, const int64_t *ro, const uint32_t *col, uint32_t *label) {
  for (int64_t v = 0; v < n; ++v) label[v] = (uint32_t)v;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      uint32_t a = uf_find(label, (uint32_t)v), b = uf_find(label, col[e]);
      if (a < b) label[b] = a;
      else if (b < a) label[a] = b;
    }
  for (int64_t v = 0; v < n; ++v) label[v] = uf_find(label, (uint32_t)v);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Betweenness centrality (traversal.py:212-278).
 * Forward sweep with path counts (forward_push_step traversal.py:121-140 with
 * accumulate_sigma): level queues ascending (np.unique), sigma of a newly
 * reached vertex = 0.0 + sum of its frontier in-neighbours' sigma in the
 * np.bincount order (queue order, then CSR order).  Direction-invariant for
 * integer-valued sigma (test_traversal.py:221-233), so the oracle pushes.
 * ------------------------------------------------------------------------- */
static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? -1 : x > y;
}

int orc_bfs_sigma(int64_t n, const int64_t *ro, const uint32_t *col, int64_t source,
                  int32_t *depth, double *sigma) {
  if (source < 0 || source >= n) return 1;
  uint32_t *q = (uint32_t *)malloc((size_t)(n + 1) * sizeof(uint32_t));
  double *add = (double *)calloc((size_t)(n ? n : 1), sizeof(double));
  if (!q || !add) { free(q); free(add); return 2; }
  for (int64_t v = 0; v < n; ++v) { depth[v] = INT32_MAX; sigma[v] = 0.0; }
  depth[source] = 0;
  sigma[source] = 1.0;
  int64_t head = 0, tail = 0;
  q[tail++] = (uint32_t)source;
  int32_t level = 0;
  while (head < tail) {
    int64_t lo = head, hi = tail;
    /* stamp the next level (unvisited destinations), queue them */
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t e = ro[q[i]]; e < ro[q[i] + 1]; ++e) {
        uint32_t v = col[e];
        if (depth[v] == INT32_MAX) { depth[v] = level + 1; q[tail++] = v; }
      }
    qsort(q + hi, (size_t)(tail - hi), sizeof(uint32_t), cmp_u32);
    /* bincount(dsts[takes], weights=sigma[srcs[takes]]) in queue x CSR order */
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t e = ro[q[i]]; e < ro[q[i] + 1]; ++e) {
        uint32_t v = col[e];
        if (depth[v] == level + 1) add[v] += sigma[q[i]];
      }
    for (int64_t i = hi; i < tail; ++i) { sigma[q[i]] += add[q[i]]; add[q[i]] = 0.0; }
    head = hi;
    ++level;
  }
  free(q);
  free(add);
  return 0;
}

/* bc_backward traversal.py:212-236: deepest level first, per vertex the
 * qualifying out-edges summed from 0.0 in CSR order, then delta += that. */
int orc_bc_backward(int64_t n, const int64_t *ro, const uint32_t *col, const int32_t *depth,
                    const double *sigma, int64_t source, double *delta) {
  int32_t maxd = -1;
  for (int64_t v = 0; v < n; ++v) {
    delta[v] = 0.0;
    if (depth[v] != INT32_MAX && depth[v] > maxd) maxd = depth[v];
  }
  for (int32_t level = maxd - 1; level >= 0; --level)
    for (int64_t v = 0; v < n; ++v) {
      if (depth[v] != level) continue;
      double acc = 0.0;
      for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
        uint32_t w = col[e];
        if (depth[w] == level + 1) acc += (sigma[v] / sigma[w]) * (1.0 + delta[w]);
      }
      delta[v] += acc;
    }
  if (source >= 0 && source < n) delta[source] = 0.0;
  return 0;
}

/* bc traversal.py:257-278: centrality += delta per source, in order. */
int orc_bc(int64_t n, const int64_t *ro, const uint32_t *col, const int64_t *sources,
           int64_t num_sources, double *centrality) {
  int32_t *depth = (int32_t *)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  double *sigma = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  double *delta = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
  if (!depth || !sigma || !delta) { free(depth); free(sigma); free(delta); return 2; }
  for (int64_t v = 0; v < n; ++v) centrality[v] = 0.0;
  int rc = 0;
  for (int64_t i = 0; i < num_sources && !rc; ++i) {
    rc = orc_bfs_sigma(n, ro, col, sources[i], depth, sigma);
    if (!rc) rc = orc_bc_backward(n, ro, col, depth, sigma, sources[i], delta);
    if (!rc)
      for (int64_t v = 0; v < n; ++v) centrality[v] += delta[v];
  }
  free(depth);
  free(sigma);
  free(delta);
  return rc;
}
