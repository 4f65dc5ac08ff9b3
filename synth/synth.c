/*
 * synth.c -- seeded, counter-based synthetic INPUT generators (weights, activations,
 * routing logits).  This module holds NONE of the method's arithmetic: it only
 * draws inputs.  It is the one piece of code that both the oracle side (tests/)
 * and the CUDA side (tests/, bench.py) consume, as DESIGN.md "Input recipe" states.
 *
 * Recipe (DESIGN.md §Input recipe, SURVEY.md §8(d) "Synthetic inputs"):
 *   hash(key, i)   = splitmix64 finaliser of key + (i+1)*golden
 *   weights        w = bf16_rn((u - 0.5) * 2 * a), u = (h >> 40) * 2^-24, a = 1/sqrt(fan_in),
 *                  0.1 % outliers (h & 1023 == 0) scaled x8 to exercise group quantisation
 *   activations    x = bf16_rn(N(0,1)) via Box-Muller on two hashes
 *   trace logits   logits[t,e] = log p_l(rank_l(e)) + Gumbel(u), p = Zipf(s) over ranks,
 *                  rank_l a seeded per-layer permutation with drift
 *
 * Built with: gcc -O2 -fPIC -shared -fopenmp (no -ffast-math).
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t hash_at(uint64_t key, uint64_t i) {
    return mix64(key + (i + 1) * 0x9e3779b97f4a7c15ULL);
}
uint64_t synth_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    uint64_t k = mix64(seed ^ 0x5bd1e9955bd1e995ULL);
    k = mix64(k ^ (a + 0x1000193ULL));
    k = mix64(k ^ (b + 0x2000327ULL));
    k = mix64(k ^ (c + 0x30004b1ULL));
    k = mix64(k ^ (d + 0x4000633ULL));
    return k;
}

static inline uint16_t f32_bf16_rn(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

/* Uniform weights with outliers; out is bf16 bits [n]. matrix id distinguishes gate/up/down/router. */
void synth_weights_bf16(uint64_t seed, int64_t layer, int64_t expert, int64_t matrix,
                        int64_t n, int64_t fan_in, uint16_t* out) {
    const uint64_t key = synth_key(seed, 1, (uint64_t)layer, (uint64_t)expert, (uint64_t)matrix);
    const float a = (float)(1.0 / sqrt((double)fan_in));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t h = hash_at(key, (uint64_t)i);
        float u = (float)(h >> 40) * (1.0f / 16777216.0f);
        float w = (u - 0.5f) * 2.0f * a;
        if ((h & 1023u) == 0) w *= 8.0f;
        out[i] = f32_bf16_rn(w);
    }
}

/* Standard-normal bf16 activations [n]. */
void synth_normal_bf16(uint64_t seed, int64_t a, int64_t b, int64_t c, int64_t n, uint16_t* out) {
    const uint64_t key = synth_key(seed, 2, (uint64_t)a, (uint64_t)b, (uint64_t)c);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t h1 = hash_at(key, 2 * (uint64_t)i), h2 = hash_at(key, 2 * (uint64_t)i + 1);
        double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        double u2 = ((double)(h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        out[i] = f32_bf16_rn((float)z);
    }
}

/* Seeded per-layer permutation rank_of[e] (expert -> popularity rank) with drift:
 * epoch 0 is a Fisher-Yates shuffle; each later epoch replaces ceil(frac * n_top) members
 * of the top-n_top ranks by swapping them with uniformly chosen ranks outside the top set
 * ("exactly ceil(rotation*|hot set|) identities change"). */
void synth_rank_perm(uint64_t seed, int64_t layer, int64_t epoch, int32_t E, int32_t n_top,
                     double frac, int32_t* rank_of) {
    int32_t* expert_at = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    uint64_t key = synth_key(seed, 3, (uint64_t)layer, 0, 0);
    for (int32_t i = 0; i < E; ++i) expert_at[i] = i;
    for (int32_t i = E - 1; i > 0; --i) {
        int32_t j = (int32_t)(hash_at(key, (uint64_t)i) % (uint64_t)(i + 1));
        int32_t tmp = expert_at[i]; expert_at[i] = expert_at[j]; expert_at[j] = tmp;
    }
    if (n_top > E) n_top = E;
    int32_t nrot = (int32_t)ceil(frac * (double)n_top);
    if (n_top >= E) nrot = 0;
    for (int64_t ep = 1; ep <= epoch; ++ep) {
        uint64_t k2 = synth_key(seed, 4, (uint64_t)layer, (uint64_t)ep, 0);
        /* choose nrot distinct positions in [0, n_top) by a partial shuffle of 0..n_top-1 */
        int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_top > 0 ? n_top : 1));
        for (int32_t i = 0; i < n_top; ++i) pos[i] = i;
        for (int32_t i = 0; i < nrot; ++i) {
            int32_t j = i + (int32_t)(hash_at(k2, (uint64_t)i) % (uint64_t)(n_top - i));
            int32_t tmp = pos[i]; pos[i] = pos[j]; pos[j] = tmp;
        }
        /* distinct outside ranks via partial shuffle of n_top..E-1 */
        int32_t nout = E - n_top;
        int32_t* out = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nout > 0 ? nout : 1));
        for (int32_t i = 0; i < nout; ++i) out[i] = n_top + i;
        for (int32_t i = 0; i < nrot && i < nout; ++i) {
            int32_t j = i + (int32_t)(hash_at(k2, 100000u + (uint64_t)i) % (uint64_t)(nout - i));
            int32_t tmp = out[i]; out[i] = out[j]; out[j] = tmp;
        }
        for (int32_t i = 0; i < nrot && i < nout; ++i) {
            int32_t a = pos[i], b = out[i];
            int32_t tmp = expert_at[a]; expert_at[a] = expert_at[b]; expert_at[b] = tmp;
        }
        free(pos); free(out);
    }
    for (int32_t r = 0; r < E; ++r) rank_of[expert_at[r]] = r;
    free(expert_at);
}

/* log-probabilities of a Zipf(s) law over ranks 0..E-1, per expert: logp[e] = log p(rank_of[e]). */
void synth_zipf_logp(const int32_t* rank_of, int32_t E, double s, float* logp) {
    double z = 0.0;
    for (int32_t r = 0; r < E; ++r) z += pow((double)(r + 1), -s);
    double lz = log(z);
    for (int32_t e = 0; e < E; ++e) logp[e] = (float)(-s * log((double)(rank_of[e] + 1)) - lz);
}

/* Trace-mode routing logits [T][E] for (layer, step): log p_l(rank(e)) + Gumbel. Top-k of these
 * is a k-draw without replacement from Zipf(s) (Gumbel-top-k). Drift epoch = step / drift_period. */
void synth_trace_logits(uint64_t seed, int64_t layer, int64_t step, int32_t T, int32_t E,
                        double zipf_s, int64_t drift_period, double drift_frac, int32_t n_top,
                        float* out) {
    int32_t* rank_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    float* logp = (float*)malloc(sizeof(float) * (size_t)E);
    int64_t epoch = drift_period > 0 ? step / drift_period : 0;
    synth_rank_perm(seed, layer, epoch, E, n_top, drift_frac, rank_of);
    synth_zipf_logp(rank_of, E, zipf_s, logp);
    const uint64_t key = synth_key(seed, 5, (uint64_t)layer, (uint64_t)step, 0);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)T * E; ++i) {
        uint64_t h = hash_at(key, (uint64_t)i);
        double u = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        double g = -log(-log(u));
        out[i] = (float)((double)logp[i % E] + g);
    }
    free(rank_of); free(logp);
}
