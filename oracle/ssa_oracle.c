/*
 * ssa_oracle.c — plain, slow, obviously-correct fp64 reference for the
 * stateful-session attention hot path of arXiv 2605.13784.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header or constant with the CUDA path
 * (paper_2605_13784_b200/csrc) and includes nothing from it.
 *
 * Every function is a direct transcription of a definition; there is no
 * tiling, fusion or reordering.  Sums run in ascending key order.
 *
 *   oracle_attention_rows   Eq. (attention), applied to
 *                           the rows of Eq. (query-attention) P:150-155 with
 *                           the causal key set of P:766 (R-2).
 *   oracle_merge_partials   split-KV log-sum-exp merge (R-11): the
 *                           softmax over a union of disjoint key sets written
 *                           as a function of the per-set (o, lse).
 *   oracle_fnv1a64          FNV-1a 64 ("FNV1a").
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

/*
 * For r in [0, nr):  the row's visible keys are keys[0 .. nvis[r]-1].
 *   s_j  = scale * sum_e q[r][e] * k[j][e]                 (QK^T / sqrt(d_k))
 *   M    = max_j s_j
 *   w_j  = exp(s_j - M),  Z = sum_j w_j                     (softmax)
 *   o[r] = sum_j w_j v[j] / Z                               (... V)
 *   lse[r] = M + log Z
 * q: [nr][d] (row stride q_stride), k: [nk][d] (stride k_stride),
 * v: [nk][dv] (stride v_stride), o: [nr][dv].  lse may be NULL.
 * A row with nvis == 0 gets o = 0, lse = -inf (empty key set, R-11).
 * Returns 0, or -1 on bad arguments / allocation failure.
 */
int oracle_attention_rows(int64_t nr, int64_t d, int64_t dv,
                          const double *q, int64_t q_stride,
                          int64_t nk, const double *k, int64_t k_stride,
                          const double *v, int64_t v_stride,
                          const int64_t *nvis, double scale,
                          double *o, double *lse)
{
    if (nr < 0 || d <= 0 || dv <= 0 || nk < 0) return -1;
    double *s = (double *)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
    if (!s) return -1;
    for (int64_t r = 0; r < nr; ++r) {
        int64_t n = nvis[r];
        if (n < 0 || n > nk) { free(s); return -1; }
        double *orow = o + r * dv;
        if (n == 0) {
            for (int64_t e = 0; e < dv; ++e) orow[e] = 0.0;
            if (lse) lse[r] = -INFINITY;
            continue;
        }
        const double *qr = q + r * q_stride;
        double m = -INFINITY;
        for (int64_t j = 0; j < n; ++j) {
            const double *kj = k + j * k_stride;
            double acc = 0.0;
            for (int64_t e = 0; e < d; ++e) acc += qr[e] * kj[e];
            s[j] = scale * acc;
            if (s[j] > m) m = s[j];
        }
        double z = 0.0;
        for (int64_t j = 0; j < n; ++j) { s[j] = exp(s[j] - m); z += s[j]; }
        for (int64_t e = 0; e < dv; ++e) {
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) acc += s[j] * v[j * v_stride + e];
            orow[e] = acc / z;
        }
        if (lse) lse[r] = m + log(z);
    }
    free(s);
    return 0;
}

/*
 * Merge G partial results of the same rows over disjoint key sets.
 * o_parts: [G][nr][dv], lse_parts: [G][nr].  For each row:
 *   L = max_g lse_g ;  w_g = exp(lse_g - L)  (w_g = 0 when lse_g = -inf)
 *   o = sum_g w_g o_g / sum_g w_g ;  lse = L + log sum_g w_g
 * All partials empty (L = -inf) -> o = 0, lse = -inf.
 */
int oracle_merge_partials(int64_t G, int64_t nr, int64_t dv,
                          const double *o_parts, const double *lse_parts,
                          double *o, double *lse)
{
    if (G <= 0 || nr < 0 || dv <= 0) return -1;
    for (int64_t r = 0; r < nr; ++r) {
        double L = -INFINITY;
        for (int64_t g = 0; g < G; ++g)
            if (lse_parts[g * nr + r] > L) L = lse_parts[g * nr + r];
        double *orow = o + r * dv;
        if (L == -INFINITY) {
            for (int64_t e = 0; e < dv; ++e) orow[e] = 0.0;
            if (lse) lse[r] = -INFINITY;
            continue;
        }
        double wsum = 0.0;
        for (int64_t g = 0; g < G; ++g) {
            double lg = lse_parts[g * nr + r];
            if (lg != -INFINITY) wsum += exp(lg - L);
        }
        for (int64_t e = 0; e < dv; ++e) {
            double acc = 0.0;
            for (int64_t g = 0; g < G; ++g) {
                double lg = lse_parts[g * nr + r];
                if (lg != -INFINITY) acc += exp(lg - L) * o_parts[(g * nr + r) * dv + e];
            }
            orow[e] = acc / wsum;
        }
        if (lse) lse[r] = L + log(wsum);
    }
    return 0;
}

/* FNV-1a, 64-bit: h = offset_basis; for each byte b: h ^= b; h *= prime. */
uint64_t oracle_fnv1a64(const uint8_t *bytes, int64_t n, uint64_t h)
{
    const uint64_t prime = 0x100000001b3ULL;
    for (int64_t i = 0; i < n; ++i) { h ^= (uint64_t)bytes[i]; h *= prime; }
    return h;
}

uint64_t oracle_fnv1a64_offset_basis(void) { return 0xcbf29ce484222325ULL; }
