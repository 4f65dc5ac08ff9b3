/*
 * oracle.c -- plain CPU oracle for DynaExq's hot path.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h).  Written from /root/reference/PAPER.md and the readings listed in
 * DESIGN.md; no blocking, fusion or reordering beyond what the definitions state.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no fast-math, no FTZ/DAZ).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ formats */
/* bf16 = upper 16 bits of an IEEE binary32 (DESIGN.md R-Q1). */
float or_bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f;
}
/* round to nearest, ties to even */
uint16_t or_f32_to_bf16_rn(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}
/* round toward +infinity (used for the stored group scale, DESIGN.md R-Q1 step 3) */
uint16_t or_f32_to_bf16_ru(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    uint16_t hi = (uint16_t)(u >> 16);
    if ((u & 0xffffu) == 0) return hi;           /* exactly representable */
    if (u >> 31) return hi;                      /* negative: truncation is toward +inf */
    return (uint16_t)(hi + 1);                   /* positive: bump magnitude (carries into exponent / inf) */
}
/* fp64 -> bf16 with a single round-to-nearest-even (no double rounding through fp32). */
uint16_t or_f64_to_bf16_rn(double d) {
    if (isnan(d)) return 0x7fc0;
    if (d == 0.0) return signbit(d) ? 0x8000 : 0x0000;
    double a = fabs(d);
    double r;
    if (a < 0x1p-126) {                          /* bf16 subnormal range: quantum 2^-133 */
        r = nearbyint(a * 0x1p133) * 0x1p-133;
    } else {
        int e; double m = frexp(a, &e);          /* a = m * 2^e, m in [0.5,1) */
        double q = nearbyint(m * 256.0);         /* 8 significant bits, RNE */
        r = ldexp(q, e - 8);
    }
    float f = (float)r;                          /* exact: r is a bf16 value (or overflows to inf) */
    if (r > 0x1.fep127) f = INFINITY;
    uint32_t u; memcpy(&u, &f, 4);
    uint16_t b = (uint16_t)(u >> 16);
    return signbit(d) ? (uint16_t)(b | 0x8000) : b;
}

/* ------------------------------------------------------------------ O-1 routing */
/* dx_expf recipe (DESIGN.md R-G2): Cody-Waite reduction + degree-7 Taylor Horner in fp32,
 * every step an exactly-rounded IEEE op, so the GPU can reproduce it bit for bit. */
float or_expf(float x) {
    if (x < -103.0f) return 0.0f;
    const float c7 = (float)(1.0 / 5040.0), c6 = (float)(1.0 / 720.0), c5 = (float)(1.0 / 120.0),
                c4 = (float)(1.0 / 24.0), c3 = (float)(1.0 / 6.0), c2 = 0.5f, c1 = 1.0f, c0 = 1.0f;
    float t = x * 0x1.715476p+0f;
    float n = rintf(t);
    float r = fmaf(n, -0x1.62e4p-1f, x);
    r = fmaf(n, -0x1.7f7d1cp-20f, r);
    float p = c7;
    p = fmaf(p, r, c6);
    p = fmaf(p, r, c5);
    p = fmaf(p, r, c4);
    p = fmaf(p, r, c3);
    p = fmaf(p, r, c2);
    p = fmaf(p, r, c1);
    p = fmaf(p, r, c0);
    return ldexpf(p, (int)n);
}

/* K = topk over logits with total order (logit desc, expert id asc); gates = softmax over the
 * k selected logits = renormalised top-k probability mass.
 * Sum is sequential in rank order in fp32; g_j = e_j / sum (IEEE division). */
int or_route(const float* logits, int32_t T, int32_t E, int32_t k, int32_t* idx, float* gate) {
    unsigned char* taken = (unsigned char*)malloc((size_t)E);
    float* ev = (float*)malloc(sizeof(float) * (size_t)k);
    int rc = 0;
    for (int32_t t = 0; t < T && rc == 0; ++t) {
        const float* l = logits + (size_t)t * E;
        /* R-G3: -inf marks a masked expert (ranked below every finite logit, gate 0 since
         * or_expf(-inf) = 0); NaN / +inf, or a token with no finite logit, violate O-1's precondition. */
        int32_t nfin = 0;
        for (int32_t e = 0; e < E; ++e) {
            if (isnan(l[e]) || (isinf(l[e]) && l[e] > 0)) rc = -1;
            nfin += isfinite(l[e]) ? 1 : 0;
            taken[e] = 0;
        }
        if (nfin == 0) rc = -1;
        if (rc) break;
        for (int32_t j = 0; j < k; ++j) {
            int32_t best = -1;
            for (int32_t e = 0; e < E; ++e) {
                if (taken[e]) continue;
                if (best < 0 || l[e] > l[best]) best = e;     /* strict '>' keeps the lower id on ties */
            }
            taken[best] = 1;
            idx[(size_t)t * k + j] = best;
        }
        float m = l[idx[(size_t)t * k]];
        float sum = 0.0f;
        for (int32_t j = 0; j < k; ++j) {
            float d = l[idx[(size_t)t * k + j]] - m;
            ev[j] = or_expf(d);
            sum = (j == 0) ? ev[0] : sum + ev[j];
        }
        for (int32_t j = 0; j < k; ++j) gate[(size_t)t * k + j] = ev[j] / sum;
    }
    free(taken); free(ev);
    return rc;
}

/* Router logits in fp64 (the router stays full precision). */
void or_router_logits(const uint16_t* x, const uint16_t* wr, const float* bias,
                      int32_t T, int32_t E, int32_t H, double* logits) {
    for (int32_t t = 0; t < T; ++t)
        for (int32_t e = 0; e < E; ++e) {
            double acc = 0.0;
            for (int32_t h = 0; h < H; ++h)
                acc += (double)or_bf16_to_f32(x[(size_t)t * H + h]) * (double)or_bf16_to_f32(wr[(size_t)e * H + h]);
            if (bias) acc += (double)bias[e];
            logits[(size_t)t * E + e] = acc;
        }
}

/* ------------------------------------------------------------------ O-2 hotness */
/* cnt_e = |{(t,j): idx = e}|, mass_e = sum of rintf(g * 2^24) (DESIGN.md R-H1).  e_lo selects the
 * local expert range [e_lo, e_lo+E) under expert parallelism. */
void or_counts(const int32_t* idx, const float* gate, int32_t n_rows, int32_t k, int32_t E,
               int32_t e_lo, uint32_t* cnt, uint64_t* mass) {
    for (int32_t e = 0; e < E; ++e) { cnt[e] = 0; mass[e] = 0; }
    for (int32_t i = 0; i < n_rows; ++i)
        for (int32_t j = 0; j < k; ++j) {
            int32_t e = idx[(size_t)i * k + j] - e_lo;
            if (e < 0 || e >= E) continue;
            cnt[e] += 1;
            mass[e] += (uint64_t)rintf(gate[(size_t)i * k + j] * 16777216.0f);
        }
}

/* Eq. 2, with Alg. 1's passive decay for experts with zero mass:
 * S <- alpha*S + (1-alpha)*gbar, gbar = mass / (B_tot * 2^24), no FMA contraction. */
void or_ema_fold(double* S, const uint64_t* mass, int32_t E, uint64_t B_tot, double alpha) {
    const double oma = 1.0 - alpha;
    const double denom = (double)B_tot * 16777216.0;
    for (int32_t e = 0; e < E; ++e) {
        double gbar = (B_tot > 0) ? (double)mass[e] / denom : 0.0;
        double a = alpha * S[e];
        double b = oma * gbar;
        S[e] = a + b;
    }
}

/* ------------------------------------------------------------------ O-3 budget */
static int64_t up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

/* Fixed-size block of one expert at `bits` ("fixed-size blocks aligned with the
 * corresponding data format"): 3 matrices of codes + bf16 scales + u8 zeros, each sub-array
 * 128 B aligned, total padded to 1024 B (DESIGN.md R-P1). */
int64_t or_slot_bytes(int32_t H, int32_t I, int32_t g, int32_t bits) {
    int64_t n = (int64_t)I * H;
    if (bits == 16) return up(3 * n * 2, 1024);
    int64_t codes = 3 * up(n * bits / 8, 128);
    int64_t sc = 2 * up((int64_t)I * (H / g) * 2, 128) + up((int64_t)H * (I / g) * 2, 128);
    int64_t zr = 2 * up((int64_t)I * (H / g), 128) + up((int64_t)H * (I / g), 128);
    return up(codes + sc + zr, 1024);
}

/* max n_hot with (n_hot+s)*S_h + (N-n_hot+s)*S_l <= M  (PAPER.md:264 inequality plus s spare
 * slots per tier, DESIGN.md R-P2).  -1 when even n_hot = 0 does not fit. */
int64_t or_n_hot(int64_t M, int32_t N, int64_t S_h, int64_t S_l, int32_t s) {
    int64_t num = M - (int64_t)N * S_l - (int64_t)s * (S_h + S_l);
    if (num < 0 || S_h <= S_l) return -1;
    int64_t n = num / (S_h - S_l);
    return n < N ? n : N;
}

/* ------------------------------------------------------------------ O-4 quantiser */
/* Asymmetric min-max RTN over groups of g consecutive elements along K (DESIGN.md R-Q1):
 *  wmin=min(0,min w), wmax=max(0,max w); s32=(wmax-wmin)/qmax; s32==0 -> 1; s=bf16_ru(s32);
 *  z=clamp(rint(-wmin/s),0,qmax); q=clamp(rint(w/s)+z,0,qmax). */
void or_quantize(const uint16_t* w, int64_t N, int64_t K, int32_t g, int32_t bits,
                 uint8_t* codes, uint16_t* scales, uint8_t* zeros) {
    const float qmax = (float)((1 << bits) - 1);
    const int64_t G = K / g;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t gi = 0; gi < G; ++gi) {
            const uint16_t* wg = w + n * K + gi * g;
            float wmin = 0.0f, wmax = 0.0f;
            for (int32_t i = 0; i < g; ++i) {
                float v = or_bf16_to_f32(wg[i]);
                if (v < wmin) wmin = v;
                if (v > wmax) wmax = v;
            }
            float s32 = (wmax - wmin) / qmax;
            if (s32 == 0.0f) s32 = 1.0f;
            uint16_t sb = or_f32_to_bf16_ru(s32);
            float s = or_bf16_to_f32(sb);
            float z = rintf(-wmin / s);
            if (z < 0.0f) z = 0.0f;
            if (z > qmax) z = qmax;
            scales[n * G + gi] = sb;
            zeros[n * G + gi] = (uint8_t)z;
            for (int32_t i = 0; i < g; ++i) {
                float q = rintf(or_bf16_to_f32(wg[i]) / s) + z;
                if (q < 0.0f) q = 0.0f;
                if (q > qmax) q = qmax;
                codes[n * K + gi * g + i] = (uint8_t)q;
            }
        }
}

/* w_hat = bf16_rn(float(q - z) * float(s)); the product is exact in fp32, one rounding. */
void or_dequantize(const uint8_t* codes, const uint16_t* scales, const uint8_t* zeros,
                   int64_t N, int64_t K, int32_t g, uint16_t* w_out) {
    const int64_t G = K / g;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t k = 0; k < K; ++k) {
            float s = or_bf16_to_f32(scales[n * G + k / g]);
            float d = (float)((int32_t)codes[n * K + k] - (int32_t)zeros[n * G + k / g]);
            w_out[n * K + k] = or_f32_to_bf16_rn(d * s);
        }
}

/* HIGH = Q_high(master) (bf16: the master itself); LOW = Q_low(deq(HIGH)) (DESIGN.md R-Q2). */
void or_expert_tier(const uint16_t* master, int32_t H, int32_t I, int32_t g,
                    int32_t high_bits, int32_t low_bits, int32_t tier_high,
                    uint16_t* w_deq, uint8_t* codes, uint16_t* scales, uint8_t* zeros) {
    const int64_t n = (int64_t)I * H;
    /* matrices: gate [I][H], up [I][H], down [H][I] */
    const int64_t rows[3] = {I, I, H}, cols[3] = {H, H, I};
    uint16_t* base = (uint16_t*)malloc(sizeof(uint16_t) * 3 * n);
    int64_t sc_off = 0;
    for (int m = 0; m < 3; ++m) {
        const uint16_t* src = master + m * n;
        uint16_t* b = base + m * n;
        if (high_bits == 16) {
            memcpy(b, src, sizeof(uint16_t) * n);
        } else {
            uint8_t* c = (uint8_t*)malloc((size_t)n);
            uint16_t* s = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(n / g));
            uint8_t* z = (uint8_t*)malloc((size_t)(n / g));
            or_quantize(src, rows[m], cols[m], g, high_bits, c, s, z);
            or_dequantize(c, s, z, rows[m], cols[m], g, b);
            if (tier_high && codes) {
                memcpy(codes + m * n, c, (size_t)n);
                memcpy(scales + sc_off, s, sizeof(uint16_t) * (size_t)(n / g));
                memcpy(zeros + sc_off, z, (size_t)(n / g));
            }
            free(c); free(s); free(z);
        }
        if (!tier_high) {
            uint8_t* c = (uint8_t*)malloc((size_t)n);
            uint16_t* s = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(n / g));
            uint8_t* z = (uint8_t*)malloc((size_t)(n / g));
            or_quantize(b, rows[m], cols[m], g, low_bits, c, s, z);
            or_dequantize(c, s, z, rows[m], cols[m], g, w_deq + m * n);
            if (codes) {
                memcpy(codes + m * n, c, (size_t)n);
                memcpy(scales + sc_off, s, sizeof(uint16_t) * (size_t)(n / g));
                memcpy(zeros + sc_off, z, (size_t)(n / g));
            }
            free(c); free(s); free(z);
        } else {
            memcpy(w_deq + m * n, b, sizeof(uint16_t) * n);
        }
        sc_off += n / g;
    }
    free(base);
}

/* ------------------------------------------------------------------ O-5 MoE FFN */
/* Routed term of Eq. 1: y = sum_{j in K} g_j(x) E_j(x), E_j a SwiGLU FFN
 *  u = Wg x, v = Wu x (fp64), a = bf16_rn(silu(u) v), o = Wd a (fp64), Y = bf16_rn(g o),
 *  y = bf16_rn(sum_j Y_j) in rank order (DESIGN.md R-F1). */
void or_moe_ffn(const uint16_t* x, const int32_t* idx, const float* gate,
                const uint16_t* const* weights, int32_t T, int32_t k, int32_t H, int32_t I,
                uint16_t* Y, uint16_t* y, int32_t nthreads) {
    const int64_t n = (int64_t)I * H;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t tj = 0; tj < (int64_t)T * k; ++tj) {
        int32_t t = (int32_t)(tj / k);
        int32_t e = idx[tj];
        const uint16_t* Wg = weights[e];
        const uint16_t* Wu = Wg + n;
        const uint16_t* Wd = Wg + 2 * n;
        const uint16_t* xt = x + (size_t)t * H;
        double* xd = (double*)malloc(sizeof(double) * (size_t)H);
        double* a = (double*)malloc(sizeof(double) * (size_t)I);
        for (int32_t h = 0; h < H; ++h) xd[h] = (double)or_bf16_to_f32(xt[h]);
        for (int32_t i = 0; i < I; ++i) {
            double u = 0.0, v = 0.0;
            for (int32_t h = 0; h < H; ++h) {
                u += (double)or_bf16_to_f32(Wg[(size_t)i * H + h]) * xd[h];
                v += (double)or_bf16_to_f32(Wu[(size_t)i * H + h]) * xd[h];
            }
            double silu = u / (1.0 + exp(-u));
            a[i] = (double)or_bf16_to_f32(or_f64_to_bf16_rn(silu * v));
        }
        for (int32_t h = 0; h < H; ++h) {
            double o = 0.0;
            for (int32_t i = 0; i < I; ++i) o += (double)or_bf16_to_f32(Wd[(size_t)h * I + i]) * a[i];
            Y[tj * H + h] = or_f64_to_bf16_rn((double)gate[tj] * o);
        }
        free(xd); free(a);
    }
    for (int32_t t = 0; t < T; ++t)
        for (int32_t h = 0; h < H; ++h) {
            double acc = 0.0;
            for (int32_t j = 0; j < k; ++j) acc += (double)or_bf16_to_f32(Y[((size_t)t * k + j) * H + h]);
            y[(size_t)t * H + h] = or_f64_to_bf16_rn(acc);
        }
}

/* ------------------------------------------------------------------ ledger */
/* alloc returns the LOWEST-index free block, -1 when exhausted. */
int32_t or_ledger_alloc(int32_t* owner, int32_t cap, int32_t who) {
    for (int32_t i = 0; i < cap; ++i) if (owner[i] < 0) { owner[i] = who; return i; }
    return -1;
}
/* free of a block not owned by `who` is ledger corruption. */
int32_t or_ledger_free(int32_t* owner, int32_t cap, int32_t slot, int32_t who) {
    if (slot < 0 || slot >= cap || owner[slot] != who) return -1;
    owner[slot] = -1;
    return 0;
}

/* ------------------------------------------------------------------ O-3/O-6 controller */
#define OR_NEVER (INT64_MIN / 4)
struct or_ctrl {
    int32_t E, n_hot, s, Tp, W, dwell, L;
    double alpha;
    int64_t t;
    double* S;
    int32_t *tier, *slot, *pend_dir, *pend_dst;
    uint32_t* version;
    int64_t *last, *pend_at;
    int32_t finalized;
    double tau;
    int32_t cap_lo, cap_hi;
    int32_t *lo_owner, *hi_owner;
};

or_ctrl* or_ctrl_create(int32_t E, int32_t n_hot, int32_t n_spare, double alpha, int32_t period,
                        int32_t warmup, int32_t dwell, int32_t lag) {
    or_ctrl* c = (or_ctrl*)calloc(1, sizeof(or_ctrl));
    c->E = E; c->n_hot = n_hot; c->s = n_spare; c->alpha = alpha; c->Tp = period; c->W = warmup;
    c->dwell = dwell; c->L = lag;
    c->S = (double*)calloc((size_t)E, sizeof(double));
    c->tier = (int32_t*)calloc((size_t)E, sizeof(int32_t));
    c->slot = (int32_t*)calloc((size_t)E, sizeof(int32_t));
    c->pend_dir = (int32_t*)calloc((size_t)E, sizeof(int32_t));
    c->pend_dst = (int32_t*)calloc((size_t)E, sizeof(int32_t));
    c->version = (uint32_t*)calloc((size_t)E, sizeof(uint32_t));
    c->last = (int64_t*)calloc((size_t)E, sizeof(int64_t));
    c->pend_at = (int64_t*)calloc((size_t)E, sizeof(int64_t));
    c->lo_owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E + n_spare));
    c->hi_owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E + n_spare));
    /* warmup layout (DESIGN.md R-P3): every expert LOW, expert e in LOW block e */
    c->cap_lo = E; c->cap_hi = 0;
    for (int32_t i = 0; i < E + n_spare; ++i) { c->lo_owner[i] = -1; c->hi_owner[i] = -1; }
    for (int32_t e = 0; e < E; ++e) { c->slot[e] = e; c->lo_owner[e] = e; c->last[e] = OR_NEVER; }
    c->tau = INFINITY;
    return c;
}

void or_ctrl_destroy(or_ctrl* c) {
    if (!c) return;
    free(c->S); free(c->tier); free(c->slot); free(c->pend_dir); free(c->pend_dst); free(c->version);
    free(c->last); free(c->pend_at); free(c->lo_owner); free(c->hi_owner); free(c);
}

/* registration + immediate reclaim of the old block, at the start of the
 * step t_plan + L (DESIGN.md R-T1) */
static void publish_due(or_ctrl* c) {
    for (int32_t e = 0; e < c->E; ++e) {
        if (c->pend_dir[e] == 0 || c->pend_at[e] != c->t) continue;
        int32_t old = c->slot[e];
        if (c->pend_dir[e] > 0) { c->lo_owner[old] = -1; c->tier[e] = 1; }
        else                    { c->hi_owner[old] = -1; c->tier[e] = 0; }
        c->slot[e] = c->pend_dst[e];
        c->version[e] += 1;
        c->pend_dir[e] = 0;
    }
}

void or_ctrl_fold(or_ctrl* c, const uint64_t* mass, uint64_t B_tot) {
    or_ema_fold(c->S, mass, c->E, B_tot, c->alpha);
    c->t += 1;
    publish_due(c);
}

/* experts in rank order: S descending, expert id ascending (SPEC.md:191 total order) */
static void rank_order(const or_ctrl* c, int32_t* order) {
    for (int32_t i = 0; i < c->E; ++i) order[i] = i;
    for (int32_t i = 1; i < c->E; ++i) {           /* insertion sort, stable on id */
        int32_t v = order[i], j = i - 1;
        while (j >= 0 && c->S[order[j]] < c->S[v]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = v;
    }
}

int32_t or_ctrl_plan(or_ctrl* c, int32_t* expert, int32_t* dir, int32_t* dst, int32_t* finalize) {
    const int32_t E = c->E;
    *finalize = 0;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    int32_t n = 0;
    if (!c->finalized && c->t == c->W) {
        /* §3.5: tau_h = top(n_hot, S) after warmup, top-n_hot initialise HIGH */
        rank_order(c, order);
        /* n_hot = N: the budget admits every expert at HIGH, no threshold applies (DESIGN.md R-C3) */
        c->tau = c->n_hot <= 0 ? INFINITY : (c->n_hot >= E ? -INFINITY : c->S[order[c->n_hot - 1]]);
        unsigned char* hot = (unsigned char*)calloc((size_t)E, 1);
        for (int32_t r = 0; r < c->n_hot; ++r) hot[order[r]] = 1;
        c->cap_lo = E - c->n_hot + c->s;
        c->cap_hi = c->n_hot + c->s;
        for (int32_t i = 0; i < E + c->s; ++i) { c->lo_owner[i] = -1; c->hi_owner[i] = -1; }
        for (int32_t e = 0; e < E; ++e)
            if (!hot[e] && c->slot[e] < c->cap_lo) c->lo_owner[c->slot[e]] = e;
        for (int32_t e = 0; e < E; ++e)
            if (!hot[e] && c->slot[e] >= c->cap_lo) {
                int32_t d = or_ledger_alloc(c->lo_owner, c->cap_lo, e);
                c->slot[e] = d;
                expert[n] = e; dir[n] = 0; dst[n] = d; ++n;
            }
        for (int32_t r = 0; r < c->n_hot; ++r) {
            int32_t e = order[r];
            c->hi_owner[r] = e; c->tier[e] = 1; c->slot[e] = r; c->version[e] += 1; c->last[e] = c->t;
            expert[n] = e; dir[n] = 1; dst[n] = r; ++n;
        }
        free(hot);
        c->finalized = 1;
        *finalize = 1;
        free(order);
        return n;
    }
    if (!c->finalized || c->t <= c->W || (c->Tp > 0 && c->t % c->Tp != 0)) { free(order); return -1; }
    for (int32_t e = 0; e < E; ++e) if (c->pend_dir[e]) { free(order); return 0; }   /* deferred */
    /* Alg. 1 PrecisionSchedule with SPEC.md:173 guards */
    rank_order(c, order);
    int32_t* P = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    int32_t* D = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    int32_t nP = 0, nD = 0, nHigh = 0;
    for (int32_t r = 0; r < E; ++r) {
        int32_t e = order[r];
        int inH = (r < c->n_hot) && (c->S[e] >= c->tau);
        if (inH && c->tier[e] == 0 && c->t - c->last[e] >= c->dwell) P[nP++] = e;
    }
    for (int32_t r = E - 1; r >= 0; --r) {
        int32_t e = order[r];
        int inH = (r < c->n_hot) && (c->S[e] >= c->tau);
        if (!inH && c->tier[e] == 1 && c->t - c->last[e] >= c->dwell) D[nD++] = e;
    }
    int32_t free_lo = 0, free_hi = 0;
    for (int32_t i = 0; i < c->cap_lo; ++i) free_lo += c->lo_owner[i] < 0;
    for (int32_t i = 0; i < c->cap_hi; ++i) free_hi += c->hi_owner[i] < 0;
    for (int32_t e = 0; e < E; ++e) nHigh += c->tier[e] == 1;
    int32_t nd = nD < free_lo ? nD : free_lo;
    int32_t np = nP < free_hi ? nP : free_hi;
    int32_t cap = c->n_hot - nHigh + nd;
    if (np > cap) np = cap;
    if (np < 0) np = 0;
    for (int32_t i = 0; i < nd; ++i) {
        int32_t e = D[i];
        int32_t d = or_ledger_alloc(c->lo_owner, c->cap_lo, e);
        c->pend_dir[e] = -1; c->pend_dst[e] = d; c->pend_at[e] = c->t + c->L; c->last[e] = c->t;
        expert[n] = e; dir[n] = -1; dst[n] = d; ++n;
    }
    for (int32_t i = 0; i < np; ++i) {
        int32_t e = P[i];
        int32_t d = or_ledger_alloc(c->hi_owner, c->cap_hi, e);
        c->pend_dir[e] = 1; c->pend_dst[e] = d; c->pend_at[e] = c->t + c->L; c->last[e] = c->t;
        expert[n] = e; dir[n] = 1; dst[n] = d; ++n;
    }
    free(P); free(D); free(order);
    return n;
}

int32_t or_ctrl_command(or_ctrl* c, int32_t e, int32_t dir) {
    if (e < 0 || e >= c->E || (dir != 1 && dir != -1)) return 2;
    if (!c->finalized) return 1;
    if (c->pend_dir[e]) return 5;
    if ((dir > 0) == (c->tier[e] == 1)) return 1;
    int32_t d = dir > 0 ? or_ledger_alloc(c->hi_owner, c->cap_hi, e)
                        : or_ledger_alloc(c->lo_owner, c->cap_lo, e);
    if (d < 0) return 4;
    c->pend_dir[e] = dir; c->pend_dst[e] = d; c->pend_at[e] = c->t + c->L; c->last[e] = c->t;
    return 0;
}

void or_ctrl_state(const or_ctrl* c, double* S, int32_t* tier, int32_t* slot, uint32_t* version,
                   int64_t* last, int32_t* in_flight, int64_t* t, double* tau,
                   int32_t* used_hi, int32_t* cap_hi, int32_t* used_lo, int32_t* cap_lo) {
    for (int32_t e = 0; e < c->E; ++e) {
        if (S) S[e] = c->S[e];
        if (tier) tier[e] = c->tier[e];
        if (slot) slot[e] = c->slot[e];
        if (version) version[e] = c->version[e];
        if (last) last[e] = c->last[e];
        if (in_flight) in_flight[e] = c->pend_dir[e];
    }
    if (t) *t = c->t;
    if (tau) *tau = c->tau;
    int32_t uh = 0, ul = 0;
    for (int32_t i = 0; i < c->cap_hi; ++i) uh += c->hi_owner[i] >= 0;
    for (int32_t i = 0; i < c->cap_lo; ++i) ul += c->lo_owner[i] >= 0;
    if (used_hi) *used_hi = uh;
    if (cap_hi) *cap_hi = c->cap_hi;
    if (used_lo) *used_lo = ul;
    if (cap_lo) *cap_lo = c->cap_lo;
}

/* TEST HOOK (unit tests of Alg. 1 on hand-built states): force a finalized
 * state with the given scores/tiers/threshold/step; HIGH experts take HIGH blocks and LOW experts
 * LOW blocks in ascending id; no transition in flight; last transition "never". */
void or_ctrl_debug_set(or_ctrl* c, const double* S, const int32_t* tier, double tau, int64_t t) {
    int32_t nlo = 0, nhi = 0;
    for (int32_t e = 0; e < c->E; ++e) { if (tier[e]) ++nhi; else ++nlo; }
    c->cap_hi = c->n_hot + c->s;
    c->cap_lo = c->E - c->n_hot + c->s;
    if (c->cap_lo < nlo) c->cap_lo = nlo;
    if (c->cap_lo > c->E + c->s) c->cap_lo = c->E + c->s;
    for (int32_t i = 0; i < c->E + c->s; ++i) { c->lo_owner[i] = -1; c->hi_owner[i] = -1; }
    for (int32_t e = 0; e < c->E; ++e) {
        c->S[e] = S[e]; c->tier[e] = tier[e] ? 1 : 0; c->pend_dir[e] = 0; c->last[e] = OR_NEVER;
        c->slot[e] = tier[e] ? or_ledger_alloc(c->hi_owner, c->cap_hi, e)
                             : or_ledger_alloc(c->lo_owner, c->cap_lo, e);
    }
    c->tau = tau; c->t = t; c->finalized = 1;
}

int32_t or_ctrl_owner(const or_ctrl* c, int32_t hi, int32_t slot) {
    if (hi) return (slot >= 0 && slot < c->cap_hi) ? c->hi_owner[slot] : -2;
    return (slot >= 0 && slot < c->cap_lo) ? c->lo_owner[slot] : -2;
}

/* ------------------------------------------------------------------ f-1 cross-layer correlation prefetch */
/* update_correlation: for every token t and every pair of an expert a chosen at
 * layer l (idx_a[t][j]) and an expert b chosen at layer l+1 (idx_b[t][j2]), corr[a][b] += 1: k*k increments
 * per token. */
void or_corr_update(uint32_t* corr, const int32_t* idx_a, const int32_t* idx_b, int32_t T, int32_t k, int32_t E) {
    for (int32_t t = 0; t < T; ++t)
        for (int32_t j = 0; j < k; ++j)
            for (int32_t j2 = 0; j2 < k; ++j2) {
                const int32_t a = idx_a[t * k + j], b = idx_b[t * k + j2];
                corr[(int64_t)a * E + b] += 1u;
            }
}

/* prefetch_candidates: up to f next-layer experts with the highest correlation to the current
 * layer's activated experts -- score(e') = sum over the T*k chosen (t, j) of corr[idx[t][j]][e'] -- filtered to
 * LOW-tier (tier 0) experts not in flight with score > 0, in (score desc, id asc) order; each paired with the next
 * lowest free HIGH block (hi_owner[b] < 0, b < cap_hi) in ascending order, so at most min(f, free blocks).
 * Returns the count. */
int32_t or_prefetch_candidates(const uint32_t* corr, const int32_t* idx, int32_t T, int32_t k, int32_t E,
                               const int32_t* tier, const int32_t* in_flight, const int32_t* hi_owner, int32_t cap_hi,
                               int32_t f, int32_t* out_e, int32_t* out_b) {
    uint64_t* score = (uint64_t*)calloc((size_t)E, sizeof(uint64_t));
    int32_t* freeb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap_hi > 0 ? cap_hi : 1));
    int32_t nfree = 0;
    for (int32_t b = 0; b < cap_hi; ++b)
        if (hi_owner[b] < 0) freeb[nfree++] = b;
    for (int32_t q = 0; q < T * k; ++q)
        for (int32_t e = 0; e < E; ++e) score[e] += corr[(int64_t)idx[q] * E + e];
    for (int32_t e = 0; e < E; ++e)
        if (tier[e] != 0 || in_flight[e] != 0) score[e] = 0;
    int32_t n = 0;
    while (n < f && n < nfree) {
        int32_t best = -1;
        for (int32_t e = 0; e < E; ++e)            /* strictly greater: ties keep the lower id */
            if (score[e] > 0 && (best < 0 || score[e] > score[best])) best = e;
        if (best < 0) break;
        out_e[n] = best;
        out_b[n] = freeb[n];
        score[best] = 0;
        ++n;
    }
    free(score);
    free(freeb);
    return n;
}

/* ------------------------------------------------------------------ f-3 shared expert (Eq. 1) */
/* The shared term of Eq. 1, y = sum_{i in S} E^s_i(x) + sum_{j in K} g_j E_j(x), with one shared expert per layer
 * (R-S1): Ys[t] = bf16_rn(E^s(x_t)), the same SwiGLU FFN and rounding points as a routed expert with gate 1
 * (u, v, o in fp64; a = bf16_rn(silu(u) v)).  W_s: the dequantised bf16 [3*I*H] image at the HIGH tier. */
void or_shared_ffn(const uint16_t* x, const uint16_t* Ws, int32_t T, int32_t H, int32_t I, uint16_t* Ys,
                   int32_t nthreads) {
    const int64_t n = (int64_t)I * H;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int32_t t = 0; t < T; ++t) {
        const uint16_t* xt = x + (size_t)t * H;
        double* xd = (double*)malloc(sizeof(double) * (size_t)H);
        double* a = (double*)malloc(sizeof(double) * (size_t)I);
        for (int32_t h = 0; h < H; ++h) xd[h] = (double)or_bf16_to_f32(xt[h]);
        for (int32_t i = 0; i < I; ++i) {
            double u = 0.0, v = 0.0;
            for (int32_t h = 0; h < H; ++h) {
                u += (double)or_bf16_to_f32(Ws[(size_t)i * H + h]) * xd[h];
                v += (double)or_bf16_to_f32(Ws[n + (size_t)i * H + h]) * xd[h];
            }
            const double silu = u / (1.0 + exp(-u));
            a[i] = (double)or_bf16_to_f32(or_f64_to_bf16_rn(silu * v));
        }
        for (int32_t h = 0; h < H; ++h) {
            double o = 0.0;
            for (int32_t i = 0; i < I; ++i) o += (double)or_bf16_to_f32(Ws[2 * n + (size_t)h * I + i]) * a[i];
            Ys[(size_t)t * H + h] = or_f64_to_bf16_rn(o);
        }
        free(xd); free(a);
    }
}
/* y[t] = bf16_rn(Ys[t] + sum_j Y[t][j]): the shared term first, then the routed rows in rank order (R-S1). */
void or_combine_shared(const uint16_t* Ys, const uint16_t* Y, int32_t T, int32_t k, int32_t H, uint16_t* y) {
    for (int32_t t = 0; t < T; ++t)
        for (int32_t h = 0; h < H; ++h) {
            double acc = (double)or_bf16_to_f32(Ys[(size_t)t * H + h]);
            for (int32_t j = 0; j < k; ++j) acc += (double)or_bf16_to_f32(Y[((size_t)t * k + j) * H + h]);
            y[(size_t)t * H + h] = or_f64_to_bf16_rn(acc);
        }
}
