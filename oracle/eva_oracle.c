/*
 * oracle/eva_oracle.c -- plain, slow, fp64 CPU oracle of the FlashEVA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2511_00576_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Citations: "P:NN" = /root/reference/PAPER.md line NN, "S:NN" = SPEC.md line NN
 * (the reference is not shipped; the lines are quoted in DESIGN.md §2).
 *
 * Everything is written in the paper's order and notation, one (batch, head)
 * unit at a time, with no blocking, fusion or reordering:
 *
 *   eps_c      ~ N(0, I_d)                 Philox4x32-10 + Box-Muller (reading R9)
 *   k~_c       = mean_{m in P_c} k_m       (Eq.10 uses k~_c; reading R1)
 *   omega_c    = lambda*clip(k~_c+eps_c)   (Eq.15, as printed; R2, R3)
 *   beta^_c    = sum_m xi(k_m,w) v_m / sum_m xi(k_m,w)   (Eq.9, S = 1)
 *                with xi(x,w) = exp(w.x - |x|^2/2)
 *   o_n        = SoftmaxAttn(q_n, K~, V~)  (Eq.12-14)
 *                K~ = {k_m : m in E(n)} U {k~_c : c < nsum(n)}
 *                V~ = {v_m : m in E(n)} U {beta^_c : c < nsum(n)}
 *
 * The one deviation from "plain": every softmax is evaluated with the row max
 * subtracted (log-domain), which is the same value in exact arithmetic; at
 * d = 128 the linear-domain xi underflows (R12).
 *
 * Beyond §8(a) (the NEXT rows of SURVEY §8(f)): the backward
 * (oracle_backward_ext, R14), the non-causal partition and summary bias (R15, R16),
 * the learned summary-key projection (oracle_summarize_proj, R17) and RoPE
 * (oracle_rope, R18) -- each written out step by step from its definition.
 *
 * Parity pins live in tests/test_oracle*.py; every function below is pinned
 * (test_oracle.py, test_oracle_backward.py, test_oracle_variants.py,
 * test_oracle_proj.py, test_oracle_rope.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: */
/* as easy as 1, 2, 3"), constants from that paper.  Pinned by the Random123  */
/* known-answer vectors in tests/golden/philox_kat.json.                       */
/* ------------------------------------------------------------------------ */
EXPORT void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                                 uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* eps for one unit (global flattened index bh = b*H + h), all nC chunks.
 * Reading R9: counter = (i, c, bh, layer) for i in [0, ceil(d/4)),
 * key = (seed_lo, seed_hi); u_j = ((x_j >> 8) + 0.5) * 2^-24 in (0, 1);
 * (z0, z1) = sqrt(-2 ln u0) * (cos, sin)(2 pi u1), (z2, z3) likewise from
 * (u2, u3); eps[c][4i + j] = z_j.  Evaluated here in fp64. */
EXPORT void oracle_eps(uint64_t seed, uint32_t layer, uint32_t bh, int nC, int d,
                       double* eps /* [nC, d] */) {
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  const double two_pi = 6.283185307179586476925286766559;
  for (int c = 0; c < nC; ++c) {
    for (int i = 0; 4 * i < d; ++i) {
      uint32_t ctr[4] = {(uint32_t)i, (uint32_t)c, bh, layer};
      uint32_t x[4];
      oracle_philox4x32_10(ctr, key, x);
      double u[4];
      for (int j = 0; j < 4; ++j) u[j] = ((double)(x[j] >> 8) + 0.5) * (1.0 / 16777216.0);
      double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
      double z[4] = {r0 * cos(two_pi * u[1]), r0 * sin(two_pi * u[1]),
                     r1 * cos(two_pi * u[3]), r1 * sin(two_pi * u[3])};
      for (int j = 0; j < 4 && 4 * i + j < d; ++j) eps[(size_t)c * d + 4 * i + j] = z[j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Partition ("local set E and disjoint subsets P_c"; P:124 custom mask; */
/* P:126 sliding window; P:298 local vs sliding variants).  0-indexed query n */
/* sees locals m in [lo, n] and summaries c < nsum.  Reading R7:               */
/*   sliding (window start quantised to a chunk boundary):             */
/*     nsum = max(0, floor(n/C) - W/C + 1), lo = nsum*C                        */
/*   block-local (original EVA, non-overlapping blocks of W):                  */
/*     lo = floor(n/W)*W, nsum = lo/C                                          */
/* ------------------------------------------------------------------------ */
EXPORT void oracle_mask(int64_t n, int C, int W, int mode, int64_t* lo, int64_t* nsum) {
  if (mode == 0) {
    int64_t s = n / C - W / C + 1;
    if (s < 0) s = 0;
    *nsum = s;
    *lo = s * C;
  } else {
    *lo = (n / W) * W;
    *nsum = *lo / C;
  }
}

/* ------------------------------------------------------------------------ */
/* Chunk summaries (Eq.9 ratio with S = 1; Eq.10     */
/* Eq.15).  For one unit: K, V are [T, d]; eps is [nC, d]; outputs [nC, d].   */
/* omega_mode 0 = Eq.15 as printed: omega = lambda * clip(k~ + eps, -1, 1)    */
/* omega_mode 1 = alternative reading: omega = k~ + lambda * clip(eps, -1, 1) */
/* ------------------------------------------------------------------------ */
static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* RoPE ("RoPE is applied to all tokens prior to the random feature projections";  */
/* NEXT row 4, DESIGN R18): rotate consecutive channel pairs (2j, 2j+1) of row x at       */
/* position pos by angle pos * base^(-2j/d):                                               */
/*   y_2j = x_2j cos a - x_2j+1 sin a,   y_2j+1 = x_2j sin a + x_2j+1 cos a.               */
/* X [T, d] in place, rows at positions pos0 .. pos0 + T - 1.                              */
EXPORT void oracle_rope(int T, int d, double base, int64_t pos0, double* X) {
  for (int t = 0; t < T; ++t) {
    double* x = X + (size_t)t * d;
    for (int j = 0; j < d / 2; ++j) {
      const double a = (double)(pos0 + t) * pow(base, -2.0 * j / (double)d);
      const double c = cos(a), s = sin(a);
      const double x0 = x[2 * j], x1 = x[2 * j + 1];
      x[2 * j] = x0 * c - x1 * s;
      x[2 * j + 1] = x0 * s + x1 * c;
    }
  }
}

/* Generalised RoPE (NEXT row 4, DESIGN R19): only the first rd channels rotate (rd even;   */
/* channels >= rd pass through, e.g. Pythia's rotary_pct), angle pos * base^(-2j/rd)  */
/* for pair j < rd/2, and the pair of j is either (2j, 2j+1) ("interleaved", style 0) or     */
/* (j, j + rd/2) (GPT-NeoX "half-split", style 1):                                          */
/*   y_a = x_a cos t - x_b sin t,   y_b = x_a sin t + x_b cos t      (a, b) = the pair j.    */
/* Row t of X [T, d] (in place) is at position pos[t].  inverse != 0: the transpose, i.e.   */
/* the rotation by -t (the gradient through RoPE).                                          */
EXPORT void oracle_rope_ex(int T, int d, double base, int rd, int style, const int64_t* pos, int inverse,
                           double* X) {
  for (int t = 0; t < T; ++t) {
    double* x = X + (size_t)t * d;
    for (int j = 0; j < rd / 2; ++j) {
      const int a = style == 0 ? 2 * j : j;
      const int b = style == 0 ? 2 * j + 1 : j + rd / 2;
      const double ang = (double)pos[t] * pow(base, -2.0 * j / (double)rd);
      const double c = cos(ang), s = inverse ? -sin(ang) : sin(ang);
      const double x0 = x[a], x1 = x[b];
      x[a] = x0 * c - x1 * s;
      x[b] = x0 * s + x1 * c;
    }
  }
}

/* P (NEXT row 4, DESIGN R17; may be NULL = identity): the learned summary-key projection,  */
/* k~_c = P (1/C) sum_i k_{cC+i} with P [d, d] row-major; mu_c = k~_c as in R2.            */
EXPORT void oracle_summarize_proj(int T, int d, int C, const double* K, const double* V,
                                  const double* eps, const double* P, double lambda, double clipv,
                                  int omega_mode, double* Ksum, double* Vsum,
                                  double* omega_out /* may be NULL */) {
  const int nC = T / C; /* trailing partial chunk is never summarised (R8) */
  double* omega = (double*)malloc(sizeof(double) * d);
  double* a = (double*)malloc(sizeof(double) * C);
  double* mean = (double*)malloc(sizeof(double) * d);
  for (int c = 0; c < nC; ++c) {
    const double* Kc = K + (size_t)c * C * d;
    const double* Vc = V + (size_t)c * C * d;
    double* kt = Ksum + (size_t)c * d;
    double* bt = Vsum + (size_t)c * d;
    /* k~_c = (1/C) sum_i k_{cC+i}  (then P k~_c when projected) */
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int i = 0; i < C; ++i) s += Kc[(size_t)i * d + j];
      mean[j] = s / (double)C;
    }
    for (int j = 0; j < d; ++j) {
      if (!P) {
        kt[j] = mean[j];
      } else {
        double s = 0.0;
        for (int l = 0; l < d; ++l) s += P[(size_t)j * d + l] * mean[l];
        kt[j] = s;
      }
    }
    /* omega_c: Eq.15 with mu_c = k~_c */
    for (int j = 0; j < d; ++j) {
      double e = eps[(size_t)c * d + j];
      if (omega_mode == 0) omega[j] = lambda * clampd(kt[j] + e, -clipv, clipv);
      else omega[j] = kt[j] + lambda * clampd(e, -clipv, clipv);
      if (omega_out) omega_out[(size_t)c * d + j] = omega[j];
    }
    /* a_i = log xi(k_i, omega) = omega . k_i - 0.5 |k_i|^2 */
    double amax = -INFINITY;
    for (int i = 0; i < C; ++i) {
      double dot = 0.0, nrm = 0.0;
      for (int j = 0; j < d; ++j) {
        double k = Kc[(size_t)i * d + j];
        dot += omega[j] * k;
        nrm += k * k;
      }
      a[i] = dot - 0.5 * nrm;
      if (a[i] > amax) amax = a[i];
    }
    /* beta^_c = sum_i softmax(a)_i v_i */
    double z = 0.0;
    for (int i = 0; i < C; ++i) z += exp(a[i] - amax);
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int i = 0; i < C; ++i) s += exp(a[i] - amax) * Vc[(size_t)i * d + j];
      bt[j] = s / z;
    }
  }
  free(omega);
  free(a);
  free(mean);
}

EXPORT void oracle_summarize(int T, int d, int C, const double* K, const double* V,
                             const double* eps, double lambda, double clipv, int omega_mode,
                             double* Ksum, double* Vsum, double* omega_out /* may be NULL */) {
  oracle_summarize_proj(T, d, C, K, V, eps, NULL, lambda, clipv, omega_mode, Ksum, Vsum, omega_out);
}

/* ------------------------------------------------------------------------ */
/* Prefill (Eq.12-14): each query is softmax attention over its    */
/* augmented key/value set.  Logit scale s multiplies q.k and q.k~ (R5).      */
/* Q, K, V, O: [T, d]; Ksum, Vsum: [nC, d]; lse: [T] (natural log).          */
/* ------------------------------------------------------------------------ */
EXPORT void oracle_prefill(int T, int d, int C, int W, int mode, double scale, const double* Q,
                           const double* K, const double* V, const double* Ksum,
                           const double* Vsum, double* O, double* lse /* may be NULL */) {
  double* logit = (double*)malloc(sizeof(double) * ((size_t)T + (size_t)T / C + 1));
  for (int n = 0; n < T; ++n) {
    int64_t lo, ns;
    oracle_mask(n, C, W, mode, &lo, &ns);
    const double* q = Q + (size_t)n * d;
    /* logits of the augmented set: summaries c < ns first, then locals lo..n */
    int cnt = 0;
    double mx = -INFINITY;
    for (int64_t c = 0; c < ns; ++c) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * Ksum[(size_t)c * d + j];
      logit[cnt] = scale * s;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    for (int64_t m = lo; m <= n; ++m) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * K[(size_t)m * d + j];
      logit[cnt] = scale * s;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    double z = 0.0;
    for (int i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
    double* o = O + (size_t)n * d;
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      int i = 0;
      for (int64_t c = 0; c < ns; ++c, ++i) acc += exp(logit[i] - mx) * Vsum[(size_t)c * d + j];
      for (int64_t m = lo; m <= n; ++m, ++i) acc += exp(logit[i] - mx) * V[(size_t)m * d + j];
      o[j] = acc / z;
    }
    if (lse) lse[n] = mx + log(z);
  }
  free(logit);
}

/* ------------------------------------------------------------------------ */
/* Prefill variants (R15, R16).            */
/*  mode 0 / 1: the causal partitions of oracle_mask (sliding / block-local). */
/*  mode 2 (non-causal, "In the non-causal setting ..."; the original   */
/*    EVA): E(n) = n's whole block of W positions [lo, min(lo+W, T)) with     */
/*    lo = floor(n/W)*W, and the summaries of every complete chunk outside    */
/*    that block, before AND after it: c < lo/C or c >= (lo+W)/C.             */
/*  bias: added to every summary logit (R16; bias = ln C counts each summary  */
/*    as the C tokens it stands for -- the |P_c| factor Eq.10 omits).   */
/* Summaries are visible as two ranges [0, s1) and [s2, nC).                   */
/* ------------------------------------------------------------------------ */
static void visible_set(int64_t n, int T, int C, int W, int mode, int64_t* lo, int64_t* hi,
                        int64_t* s1, int64_t* s2) {
  const int64_t nC = T / C;
  if (mode == 2) {
    *lo = (n / W) * W;
    *hi = *lo + W < T ? *lo + W : T;
    *s1 = *lo / C;
    *s2 = (*lo + W) / C;
    if (*s2 > nC) *s2 = nC;
  } else {
    int64_t ns;
    oracle_mask(n, C, W, mode, lo, &ns);
    *hi = n + 1;
    *s1 = ns;
    *s2 = nC;
  }
}

EXPORT void oracle_prefill_ext(int T, int d, int C, int W, int mode, double scale, double bias,
                               const double* Q, const double* K, const double* V,
                               const double* Ksum, const double* Vsum, double* O,
                               double* lse /* may be NULL */) {
  const int64_t nC = T / C;
  double* logit = (double*)malloc(sizeof(double) * ((size_t)T + (size_t)nC + 1));
  for (int n = 0; n < T; ++n) {
    int64_t lo, hi, s1, s2;
    visible_set(n, T, C, W, mode, &lo, &hi, &s1, &s2);
    const double* q = Q + (size_t)n * d;
    int cnt = 0;
    double mx = -INFINITY;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * Ksum[(size_t)c * d + j];
      logit[cnt] = scale * s + bias;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    for (int64_t m = lo; m < hi; ++m) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * K[(size_t)m * d + j];
      logit[cnt] = scale * s;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    double z = 0.0;
    for (int i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
    double* o = O + (size_t)n * d;
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      int i = 0;
      for (int64_t c = 0; c < nC; ++c) {
        if (!(c < s1 || c >= s2)) continue;
        acc += exp(logit[i++] - mx) * Vsum[(size_t)c * d + j];
      }
      for (int64_t m = lo; m < hi; ++m) acc += exp(logit[i++] - mx) * V[(size_t)m * d + j];
      o[j] = acc / z;
    }
    if (lse) lse[n] = mx + log(z);
  }
  free(logit);
}

EXPORT void oracle_prefill_ext_batch(int BH, int T, int d, int C, int W, int mode, double scale,
                                     double bias, const double* Q, const double* K, const double* V,
                                     const double* Ksum, const double* Vsum, double* O, double* lse) {
  const int nC = T / C;
#pragma omp parallel for schedule(dynamic, 1)
  for (int u = 0; u < BH; ++u)
    oracle_prefill_ext(T, d, C, W, mode, scale, bias, Q + (size_t)u * T * d, K + (size_t)u * T * d,
                       V + (size_t)u * T * d, Ksum + (size_t)u * nC * d, Vsum + (size_t)u * nC * d,
                       O + (size_t)u * T * d, lse ? lse + (size_t)u * T : NULL);
}

/* ------------------------------------------------------------------------ */
/* Batched drivers: the same per-unit functions over BH units.  The loop is   */
/* over independent units only (no change to any unit's arithmetic).          */
/* ------------------------------------------------------------------------ */
EXPORT void oracle_summarize_batch(int BH, int T, int d, int C, const double* K, const double* V,
                                   const double* eps, double lambda, double clipv, int omega_mode,
                                   double* Ksum, double* Vsum) {
  const int nC = T / C;
#pragma omp parallel for schedule(dynamic, 1)
  for (int u = 0; u < BH; ++u)
    oracle_summarize(T, d, C, K + (size_t)u * T * d, V + (size_t)u * T * d,
                     eps + (size_t)u * nC * d, lambda, clipv, omega_mode,
                     Ksum + (size_t)u * nC * d, Vsum + (size_t)u * nC * d, NULL);
}

EXPORT void oracle_prefill_batch(int BH, int T, int d, int C, int W, int mode, double scale,
                                 const double* Q, const double* K, const double* V,
                                 const double* Ksum, const double* Vsum, double* O, double* lse) {
  const int nC = T / C;
#pragma omp parallel for schedule(dynamic, 1)
  for (int u = 0; u < BH; ++u)
    oracle_prefill(T, d, C, W, mode, scale, Q + (size_t)u * T * d, K + (size_t)u * T * d,
                   V + (size_t)u * T * d, Ksum + (size_t)u * nC * d, Vsum + (size_t)u * nC * d,
                   O + (size_t)u * T * d, lse ? lse + (size_t)u * T : NULL);
}

/* Prefill for a subset of query rows (large-size sampled parity): rows[r]    */
/* are query indices; O_rows [R, d], lse_rows [R].  Same row formula.          */
EXPORT void oracle_prefill_rows(int T, int d, int C, int W, int mode, double scale,
                                const double* Q, const double* K, const double* V,
                                const double* Ksum, const double* Vsum, int R,
                                const int64_t* rows, double* O_rows, double* lse_rows) {
  (void)T;
  double* logit = (double*)malloc(sizeof(double) * ((size_t)W + (size_t)rows[R - 1] / C + 2));
  for (int r = 0; r < R; ++r) {
    int64_t n = rows[r], lo, ns;
    oracle_mask(n, C, W, mode, &lo, &ns);
    const double* q = Q + (size_t)n * d;
    int cnt = 0;
    double mx = -INFINITY;
    for (int64_t c = 0; c < ns; ++c) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * Ksum[(size_t)c * d + j];
      logit[cnt] = scale * s;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    for (int64_t m = lo; m <= n; ++m) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += q[j] * K[(size_t)m * d + j];
      logit[cnt] = scale * s;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    double z = 0.0;
    for (int i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      int i = 0;
      for (int64_t c = 0; c < ns; ++c, ++i) acc += exp(logit[i] - mx) * Vsum[(size_t)c * d + j];
      for (int64_t m = lo; m <= n; ++m, ++i) acc += exp(logit[i] - mx) * V[(size_t)m * d + j];
      O_rows[(size_t)r * d + j] = acc / z;
    }
    if (lse_rows) lse_rows[r] = mx + log(z);
  }
  free(logit);
}

/* ------------------------------------------------------------------------ */
/* Streaming decode with the compressed cache ("cache of          */
/* (compressed) past context").  One unit.  The state after        */
/* positions 0..pos-1 holds a ring of the last W (k, v) pairs (slot p mod W)  */
/* and every completed chunk's summary.  A chunk is summarised when its last  */
/* token arrives (eager; equivalent to SPEC's lazy compress-on-eviction,      */
/* S:359, because a summary depends only on its own chunk and eps_c, R13).    */
/* ------------------------------------------------------------------------ */
typedef struct {
  int d, C, W, mode, cap;
  double scale, lambda, clipv;
  int omega_mode;
  int64_t pos;
  double *ring_k, *ring_v; /* [W, d] */
  double *sum_k, *sum_v;   /* [cap, d] */
} oracle_cache;

EXPORT oracle_cache* oracle_cache_new(int d, int C, int W, int mode, int cap, double scale,
                                      double lambda, double clipv, int omega_mode) {
  oracle_cache* s = (oracle_cache*)calloc(1, sizeof(oracle_cache));
  s->d = d; s->C = C; s->W = W; s->mode = mode; s->cap = cap;
  s->scale = scale; s->lambda = lambda; s->clipv = clipv; s->omega_mode = omega_mode;
  s->pos = 0;
  s->ring_k = (double*)calloc((size_t)W * d, sizeof(double));
  s->ring_v = (double*)calloc((size_t)W * d, sizeof(double));
  s->sum_k = (double*)calloc((size_t)cap * d, sizeof(double));
  s->sum_v = (double*)calloc((size_t)cap * d, sizeof(double));
  return s;
}

EXPORT void oracle_cache_free(oracle_cache* s) {
  if (!s) return;
  free(s->ring_k); free(s->ring_v); free(s->sum_k); free(s->sum_v); free(s);
}

EXPORT int64_t oracle_cache_pos(const oracle_cache* s) { return s->pos; }
EXPORT const double* oracle_cache_sum_k(const oracle_cache* s) { return s->sum_k; }
EXPORT const double* oracle_cache_sum_v(const oracle_cache* s) { return s->sum_v; }

/* Append one token (k, v) at position pos.  eps_chunk is eps of the chunk   */
/* pos/C ([d]); it is read only when this token completes the chunk.         */
/* Returns 0, or 3 when the summary list is full (capacity error).           */
EXPORT int oracle_cache_append(oracle_cache* s, const double* k, const double* v,
                               const double* eps_chunk) {
  const int d = s->d, C = s->C, W = s->W;
  const int64_t p = s->pos;
  if ((p + 1) % C == 0 && (p + 1) / C > s->cap) return 3;
  memcpy(s->ring_k + (size_t)(p % W) * d, k, sizeof(double) * d);
  memcpy(s->ring_v + (size_t)(p % W) * d, v, sizeof(double) * d);
  if ((p + 1) % C == 0) {
    /* the chunk [p+1-C, p] is entirely in the ring (W >= C): gather it */
    const int64_t c = (p + 1) / C - 1;
    double* Kc = (double*)malloc(sizeof(double) * (size_t)C * d);
    double* Vc = (double*)malloc(sizeof(double) * (size_t)C * d);
    for (int i = 0; i < C; ++i) {
      int64_t q = c * C + i;
      memcpy(Kc + (size_t)i * d, s->ring_k + (size_t)(q % W) * d, sizeof(double) * d);
      memcpy(Vc + (size_t)i * d, s->ring_v + (size_t)(q % W) * d, sizeof(double) * d);
    }
    oracle_summarize(C, d, C, Kc, Vc, eps_chunk, s->lambda, s->clipv, s->omega_mode,
                     s->sum_k + (size_t)c * d, s->sum_v + (size_t)c * d, NULL);
    free(Kc);
    free(Vc);
  }
  s->pos = p + 1;
  return 0;
}

/* Attend query q (the token at position pos-1) over the cache (Eq.12 for a   */
/* single query).  o: [d]; returns lse.                                       */
EXPORT double oracle_cache_decode(const oracle_cache* s, const double* q, double* o) {
  const int d = s->d, C = s->C, W = s->W;
  const int64_t n = s->pos - 1;
  int64_t lo, ns;
  oracle_mask(n, C, W, s->mode, &lo, &ns);
  const int64_t cnt = ns + (n - lo + 1);
  double* logit = (double*)malloc(sizeof(double) * (size_t)cnt);
  double mx = -INFINITY;
  int64_t i = 0;
  for (int64_t c = 0; c < ns; ++c, ++i) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t += q[j] * s->sum_k[(size_t)c * d + j];
    logit[i] = s->scale * t;
    if (logit[i] > mx) mx = logit[i];
  }
  for (int64_t m = lo; m <= n; ++m, ++i) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t += q[j] * s->ring_k[(size_t)(m % W) * d + j];
    logit[i] = s->scale * t;
    if (logit[i] > mx) mx = logit[i];
  }
  double z = 0.0;
  for (i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
  for (int j = 0; j < d; ++j) {
    double acc = 0.0;
    i = 0;
    for (int64_t c = 0; c < ns; ++c, ++i) acc += exp(logit[i] - mx) * s->sum_v[(size_t)c * d + j];
    for (int64_t m = lo; m <= n; ++m, ++i)
      acc += exp(logit[i] - mx) * s->ring_v[(size_t)(m % W) * d + j];
    o[j] = acc / z;
  }
  free(logit);
  return mx + log(z);
}

/* ------------------------------------------------------------------------ */
/* Backward of the prefill (NEXT row 1: the paper's training path,    */
/* P:253 "forward and backward pass").  For L = sum_n dO_n . o_n it returns  */
/* dQ, dK, dV of one unit, written out step by step from the forward:       */
/*  attention (Eq.12): P_nx = softmax_x(s q_n.key_x), D_n = dO_n . o_n,      */
/*    dS_nx = P_nx (dO_n . val_x - D_n); dq_n = s sum_x dS_nx key_x;         */
/*    local x = m: dk_m += s dS_nm q_n, dv_m += P_nm dO_n;                   */
/*    summary x = c: dk~_c += s dS_nc q_n, dbeta_c += P_nc dO_n.             */
/*  summaries (Eq.9, Eq.10, Eq.15), chunk c with rows i:           */
/*    w_i = softmax_i(a_i), a_i = omega.k_i - |k_i|^2/2, beta = sum w_i v_i:  */
/*    dv_i += w_i dbeta; da_i = w_i (dbeta.v_i - dbeta.beta);                */
/*    dk_i += da_i (omega - k_i); domega = sum_i da_i k_i;                    */
/*    omega = lambda clip(k~ + eps): dk~ += lambda [|k~+eps| <= clip] domega  */
/*    (as printed; the shifted reading omega = k~ + lambda clip(eps) gives    */
/*    dk~ += domega); k~ = mean k_i: dk_i += dk~ / C.                         */
/* eps is a constant.  Q, K, V, dO, dQ, dK, dV: [T, d]; eps [nC, d].          */
/* ------------------------------------------------------------------------ */
/* The variants (DESIGN R15, R16) change only the visible sets and the summary logits:    */
/* summary c visible iff c < s1 or c >= s2, locals [lo, hi) (visible_set), and the summary  */
/* logit is s q.k~_c + bias.  The bias is a constant, so dS / dk~ / dbeta keep their form.  */
EXPORT void oracle_backward_ext(int T, int d, int C, int W, int mode, double scale, double bias,
                                double lambda, double clipv, int omega_mode, const double* Q,
                                const double* K, const double* V, const double* eps,
                                const double* dO, double* dQ, double* dK, double* dV) {
  const int nC = T / C;
  const size_t nd = (size_t)(nC > 0 ? nC : 1) * d;
  double* kt = (double*)calloc(nd, sizeof(double));
  double* bt = (double*)calloc(nd, sizeof(double));
  double* om = (double*)calloc(nd, sizeof(double));
  double* dkt = (double*)calloc(nd, sizeof(double));
  double* dbt = (double*)calloc(nd, sizeof(double));
  double* logit = (double*)malloc(sizeof(double) * ((size_t)T + nC + 1));
  double* o = (double*)malloc(sizeof(double) * d);
  if (nC > 0) oracle_summarize(T, d, C, K, V, eps, lambda, clipv, omega_mode, kt, bt, om);
  memset(dQ, 0, sizeof(double) * (size_t)T * d);
  memset(dK, 0, sizeof(double) * (size_t)T * d);
  memset(dV, 0, sizeof(double) * (size_t)T * d);
  for (int n = 0; n < T; ++n) {
    int64_t lo, hi, s1, s2;
    visible_set(n, T, C, W, mode, &lo, &hi, &s1, &s2);
    const double* q = Q + (size_t)n * d;
    const double* g = dO + (size_t)n * d;
    int cnt = 0;
    double mx = -INFINITY;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      double t = 0.0;
      for (int j = 0; j < d; ++j) t += q[j] * kt[(size_t)c * d + j];
      logit[cnt] = scale * t + bias;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    for (int64_t m = lo; m < hi; ++m, ++cnt) {
      double t = 0.0;
      for (int j = 0; j < d; ++j) t += q[j] * K[(size_t)m * d + j];
      logit[cnt] = scale * t;
      if (logit[cnt] > mx) mx = logit[cnt];
    }
    double z = 0.0;
    for (int i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
    for (int i = 0; i < cnt; ++i) logit[i] = exp(logit[i] - mx) / z; /* now P */
    for (int j = 0; j < d; ++j) o[j] = 0.0;
    int i = 0;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      for (int j = 0; j < d; ++j) o[j] += logit[i] * bt[(size_t)c * d + j];
      ++i;
    }
    for (int64_t m = lo; m < hi; ++m, ++i)
      for (int j = 0; j < d; ++j) o[j] += logit[i] * V[(size_t)m * d + j];
    double Dn = 0.0;
    for (int j = 0; j < d; ++j) Dn += g[j] * o[j];
    i = 0;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      double dp = 0.0;
      for (int j = 0; j < d; ++j) dp += g[j] * bt[(size_t)c * d + j];
      const double dS = logit[i] * (dp - Dn);
      for (int j = 0; j < d; ++j) {
        dQ[(size_t)n * d + j] += scale * dS * kt[(size_t)c * d + j];
        dkt[(size_t)c * d + j] += scale * dS * q[j];
        dbt[(size_t)c * d + j] += logit[i] * g[j];
      }
      ++i;
    }
    for (int64_t m = lo; m < hi; ++m, ++i) {
      double dp = 0.0;
      for (int j = 0; j < d; ++j) dp += g[j] * V[(size_t)m * d + j];
      const double dS = logit[i] * (dp - Dn);
      for (int j = 0; j < d; ++j) {
        dQ[(size_t)n * d + j] += scale * dS * K[(size_t)m * d + j];
        dK[(size_t)m * d + j] += scale * dS * q[j];
        dV[(size_t)m * d + j] += logit[i] * g[j];
      }
    }
  }
  /* through the summaries */
  double* a = (double*)malloc(sizeof(double) * (C > 0 ? C : 1));
  double* dom = (double*)malloc(sizeof(double) * d);
  for (int c = 0; c < nC; ++c) {
    const double* Kc = K + (size_t)c * C * d;
    const double* Vc = V + (size_t)c * C * d;
    const double* w_om = om + (size_t)c * d;
    const double* db = dbt + (size_t)c * d;
    const double* be = bt + (size_t)c * d;
    double amax = -INFINITY;
    for (int r = 0; r < C; ++r) {
      double dot = 0.0, nrm = 0.0;
      for (int j = 0; j < d; ++j) {
        dot += w_om[j] * Kc[(size_t)r * d + j];
        nrm += Kc[(size_t)r * d + j] * Kc[(size_t)r * d + j];
      }
      a[r] = dot - 0.5 * nrm;
      if (a[r] > amax) amax = a[r];
    }
    double zz = 0.0;
    for (int r = 0; r < C; ++r) zz += exp(a[r] - amax);
    double dbb = 0.0;
    for (int j = 0; j < d; ++j) dbb += db[j] * be[j];
    for (int j = 0; j < d; ++j) dom[j] = 0.0;
    for (int r = 0; r < C; ++r) {
      const double w = exp(a[r] - amax) / zz;
      double dbv = 0.0;
      for (int j = 0; j < d; ++j) dbv += db[j] * Vc[(size_t)r * d + j];
      const double da = w * (dbv - dbb);
      for (int j = 0; j < d; ++j) {
        dV[((size_t)c * C + r) * d + j] += w * db[j];
        dK[((size_t)c * C + r) * d + j] += da * (w_om[j] - Kc[(size_t)r * d + j]);
        dom[j] += da * Kc[(size_t)r * d + j];
      }
    }
    for (int j = 0; j < d; ++j) {
      double dk_t = dkt[(size_t)c * d + j];
      if (omega_mode == 0) {
        const double x = kt[(size_t)c * d + j] + eps[(size_t)c * d + j];
        if (x >= -clipv && x <= clipv) dk_t += lambda * dom[j];
      } else {
        dk_t += dom[j];
      }
      for (int r = 0; r < C; ++r) dK[((size_t)c * C + r) * d + j] += dk_t / (double)C;
    }
  }
  free(a); free(dom); free(kt); free(bt); free(om); free(dkt); free(dbt); free(logit); free(o);
}

/* Backward with the learned summary-key projection (NEXT row 4, DESIGN R17): the forward is  */
/* oracle_summarize_proj (k~_c = P mean_c, mu_c = k~_c in Eq.15, xi from the raw keys) and     */
/* oracle_prefill on (k~, beta^).  The attention part is oracle_backward_ext's (causal modes,  */
/* no bias); through the summaries, per chunk c with dk~ from the attention and d beta^:       */
/*   dv_i += w_i d beta^;  da_i = w_i (d beta^ . v_i - d beta^ . beta^);                      */
/*   dk_i += da_i (omega - k_i);  d omega = sum_i da_i k_i;                                   */
/*   g_j = d k~_j + lambda [|k~_j + eps_j| <= clip] d omega_j   (omega_mode 1: + d omega_j);  */
/*   k~ = P mean:  d mean = P^T g,  dk_i += d mean / C,  dP += g mean^T.                       */
/* P [d, d] row-major; dP [d, d] is ACCUMULATED (the caller zeroes it).                        */
EXPORT void oracle_backward_proj(int T, int d, int C, int W, int mode, double scale, double lambda,
                                 double clipv, int omega_mode, const double* Q, const double* K,
                                 const double* V, const double* eps, const double* P, const double* dO,
                                 double* dQ, double* dK, double* dV, double* dP) {
  const int nC = T / C;
  const size_t nd = (size_t)(nC > 0 ? nC : 1) * d;
  double* kt = (double*)calloc(nd, sizeof(double));
  double* bt = (double*)calloc(nd, sizeof(double));
  double* om = (double*)calloc(nd, sizeof(double));
  double* dkt = (double*)calloc(nd, sizeof(double));
  double* dbt = (double*)calloc(nd, sizeof(double));
  double* logit = (double*)malloc(sizeof(double) * ((size_t)T + nC + 1));
  double* o = (double*)malloc(sizeof(double) * d);
  if (nC > 0) oracle_summarize_proj(T, d, C, K, V, eps, P, lambda, clipv, omega_mode, kt, bt, om);
  memset(dQ, 0, sizeof(double) * (size_t)T * d);
  memset(dK, 0, sizeof(double) * (size_t)T * d);
  memset(dV, 0, sizeof(double) * (size_t)T * d);
  for (int n = 0; n < T; ++n) {  /* the attention: softmax over the summaries and the window */
    int64_t lo, hi, s1, s2;
    visible_set(n, T, C, W, mode, &lo, &hi, &s1, &s2);
    const double* q = Q + (size_t)n * d;
    const double* g = dO + (size_t)n * d;
    int cnt = 0;
    double mx = -INFINITY;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      double t = 0.0;
      for (int j = 0; j < d; ++j) t += q[j] * kt[(size_t)c * d + j];
      logit[cnt] = scale * t;
      if (logit[cnt] > mx) mx = logit[cnt];
      ++cnt;
    }
    for (int64_t m = lo; m < hi; ++m, ++cnt) {
      double t = 0.0;
      for (int j = 0; j < d; ++j) t += q[j] * K[(size_t)m * d + j];
      logit[cnt] = scale * t;
      if (logit[cnt] > mx) mx = logit[cnt];
    }
    double z = 0.0;
    for (int i = 0; i < cnt; ++i) z += exp(logit[i] - mx);
    for (int i = 0; i < cnt; ++i) logit[i] = exp(logit[i] - mx) / z;
    for (int j = 0; j < d; ++j) o[j] = 0.0;
    int i = 0;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      for (int j = 0; j < d; ++j) o[j] += logit[i] * bt[(size_t)c * d + j];
      ++i;
    }
    for (int64_t m = lo; m < hi; ++m, ++i)
      for (int j = 0; j < d; ++j) o[j] += logit[i] * V[(size_t)m * d + j];
    double Dn = 0.0;
    for (int j = 0; j < d; ++j) Dn += g[j] * o[j];
    i = 0;
    for (int64_t c = 0; c < nC; ++c) {
      if (!(c < s1 || c >= s2)) continue;
      double dp = 0.0;
      for (int j = 0; j < d; ++j) dp += g[j] * bt[(size_t)c * d + j];
      const double dS = logit[i] * (dp - Dn);
      for (int j = 0; j < d; ++j) {
        dQ[(size_t)n * d + j] += scale * dS * kt[(size_t)c * d + j];
        dkt[(size_t)c * d + j] += scale * dS * q[j];
        dbt[(size_t)c * d + j] += logit[i] * g[j];
      }
      ++i;
    }
    for (int64_t m = lo; m < hi; ++m, ++i) {
      double dp = 0.0;
      for (int j = 0; j < d; ++j) dp += g[j] * V[(size_t)m * d + j];
      const double dS = logit[i] * (dp - Dn);
      for (int j = 0; j < d; ++j) {
        dQ[(size_t)n * d + j] += scale * dS * K[(size_t)m * d + j];
        dK[(size_t)m * d + j] += scale * dS * q[j];
        dV[(size_t)m * d + j] += logit[i] * g[j];
      }
    }
  }
  double* a = (double*)malloc(sizeof(double) * (C > 0 ? C : 1));
  double* dom = (double*)malloc(sizeof(double) * d);
  double* gk = (double*)malloc(sizeof(double) * d);
  double* mean = (double*)malloc(sizeof(double) * d);
  for (int c = 0; c < nC; ++c) {  /* through the summaries of chunk c */
    const double* Kc = K + (size_t)c * C * d;
    const double* Vc = V + (size_t)c * C * d;
    const double* w_om = om + (size_t)c * d;
    const double* db = dbt + (size_t)c * d;
    const double* be = bt + (size_t)c * d;
    for (int j = 0; j < d; ++j) {
      mean[j] = 0.0;
      for (int r = 0; r < C; ++r) mean[j] += Kc[(size_t)r * d + j];
      mean[j] /= (double)C;
    }
    double amax = -INFINITY;
    for (int r = 0; r < C; ++r) {
      double dot = 0.0, nrm = 0.0;
      for (int j = 0; j < d; ++j) {
        dot += w_om[j] * Kc[(size_t)r * d + j];
        nrm += Kc[(size_t)r * d + j] * Kc[(size_t)r * d + j];
      }
      a[r] = dot - 0.5 * nrm;
      if (a[r] > amax) amax = a[r];
    }
    double zz = 0.0;
    for (int r = 0; r < C; ++r) zz += exp(a[r] - amax);
    double dbb = 0.0;
    for (int j = 0; j < d; ++j) dbb += db[j] * be[j];
    for (int j = 0; j < d; ++j) dom[j] = 0.0;
    for (int r = 0; r < C; ++r) {
      const double w = exp(a[r] - amax) / zz;
      double dbv = 0.0;
      for (int j = 0; j < d; ++j) dbv += db[j] * Vc[(size_t)r * d + j];
      const double da = w * (dbv - dbb);
      for (int j = 0; j < d; ++j) {
        dV[((size_t)c * C + r) * d + j] += w * db[j];
        dK[((size_t)c * C + r) * d + j] += da * (w_om[j] - Kc[(size_t)r * d + j]);
        dom[j] += da * Kc[(size_t)r * d + j];
      }
    }
    for (int j = 0; j < d; ++j) {  /* g = total gradient of k~_c */
      gk[j] = dkt[(size_t)c * d + j];
      if (omega_mode == 0) {
        const double x = kt[(size_t)c * d + j] + eps[(size_t)c * d + j];
        if (x >= -clipv && x <= clipv) gk[j] += lambda * dom[j];
      } else {
        gk[j] += dom[j];
      }
    }
    for (int l = 0; l < d; ++l) {  /* d mean = P^T g, spread over the chunk's rows; dP += g mean^T */
      double dm = 0.0;
      for (int j = 0; j < d; ++j) dm += (P ? P[(size_t)j * d + l] : (j == l ? 1.0 : 0.0)) * gk[j];
      for (int r = 0; r < C; ++r) dK[((size_t)c * C + r) * d + l] += dm / (double)C;
    }
    if (dP)
      for (int j = 0; j < d; ++j)
        for (int l = 0; l < d; ++l) dP[(size_t)j * d + l] += gk[j] * mean[l];
  }
  free(a); free(dom); free(gk); free(mean); free(kt); free(bt); free(om); free(dkt); free(dbt);
  free(logit); free(o);
}

EXPORT void oracle_backward(int T, int d, int C, int W, int mode, double scale, double lambda,
                            double clipv, int omega_mode, const double* Q, const double* K,
                            const double* V, const double* eps, const double* dO, double* dQ,
                            double* dK, double* dV) {
  oracle_backward_ext(T, d, C, W, mode, scale, 0.0, lambda, clipv, omega_mode, Q, K, V, eps, dO,
                      dQ, dK, dV);
}

EXPORT void oracle_backward_ext_batch(int BH, int T, int d, int C, int W, int mode, double scale,
                                      double bias, double lambda, double clipv, int omega_mode,
                                      const double* Q, const double* K, const double* V,
                                      const double* eps, const double* dO, double* dQ,
                                      double* dK, double* dV) {
  const int nC = T / C;
#pragma omp parallel for schedule(dynamic, 1)
  for (int u = 0; u < BH; ++u) {
    const size_t off = (size_t)u * T * d;
    oracle_backward_ext(T, d, C, W, mode, scale, bias, lambda, clipv, omega_mode, Q + off, K + off,
                        V + off, eps + (size_t)u * nC * d, dO + off, dQ + off, dK + off, dV + off);
  }
}

EXPORT void oracle_backward_batch(int BH, int T, int d, int C, int W, int mode, double scale,
                                  double lambda, double clipv, int omega_mode, const double* Q,
                                  const double* K, const double* V, const double* eps,
                                  const double* dO, double* dQ, double* dK, double* dV) {
  oracle_backward_ext_batch(BH, T, d, C, W, mode, scale, 0.0, lambda, clipv, omega_mode, Q, K, V,
                            eps, dO, dQ, dK, dV);
}
