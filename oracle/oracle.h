/*
 * oracle.h -- plain, slow, obviously-correct CPU ORACLE for DynaExq's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2511_15015_b200/) never imports, links or executes anything under oracle/,
 * and shares no code with it (no headers, helpers, tables or constants).
 *
 * Every function cites the passage of /root/reference/PAPER.md (or SPEC.md, or the
 * DESIGN.md reading where the paper is silent) that it follows.  Floating point is
 * fp64 except where the method fixes fp32/bf16.  Built with
 * gcc -O2 -ffp-contract=off, no fast-math, so fmaf/rintf/ldexpf/division are IEEE.
 *
 * Parity status of each function is stated in DESIGN.md "Oracle pins".
 */
#ifndef DYNAEXQ_ORACLE_H
#define DYNAEXQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- numeric formats (DESIGN.md R-Q1) ---- */
float    or_bf16_to_f32(uint16_t b);
uint16_t or_f32_to_bf16_rn(float f);
uint16_t or_f32_to_bf16_ru(float f);
uint16_t or_f64_to_bf16_rn(double d);

/* ---- O-1 router, top-k, gates (Eq.1 "K = topk({g_i(x)})") ---- */
float or_expf(float x);                                   /* DESIGN.md R-G2 recipe, x <= 0 */
int   or_route(const float* logits, int32_t T, int32_t E, int32_t k,
               int32_t* idx, float* gate);                /* 0 ok, -1 NaN/+inf or no finite logit (R-G3) */
void  or_router_logits(const uint16_t* x, const uint16_t* wr, const float* bias,
                       int32_t T, int32_t E, int32_t H, double* logits);

/* ---- O-2 hotness counters and EMA ("records the selected experts and
 *      accumulates gating probabilities"; Eq. 2; Alg.1) ---- */
void or_counts(const int32_t* idx, const float* gate, int32_t n_rows, int32_t k, int32_t E,
               int32_t e_lo, uint32_t* cnt, uint64_t* mass);
void or_ema_fold(double* S, const uint64_t* mass, int32_t E, uint64_t B_tot, double alpha);

/* ---- O-3 budget (§3.5) ---- */
int64_t or_slot_bytes(int32_t H, int32_t I, int32_t g, int32_t bits);
int64_t or_n_hot(int64_t M, int32_t N, int64_t S_h, int64_t S_l, int32_t s); /* -1 infeasible */

/* ---- O-4 group quantiser (PAPER.md:274 AutoRound; :253 "FP16 or INT4"; DESIGN.md R-Q1) ---- */
void or_quantize(const uint16_t* w, int64_t N, int64_t K, int32_t g, int32_t bits,
                 uint8_t* codes, uint16_t* scales, uint8_t* zeros);
void or_dequantize(const uint8_t* codes, const uint16_t* scales, const uint8_t* zeros,
                   int64_t N, int64_t K, int32_t g, uint16_t* w_out);
/* canonical image of one expert at `bits` (16: copy of master); path independence:
 * LOW = Q_low(deq(HIGH)), HIGH = Q_high(master) (DESIGN.md R-Q2).  Returns the
 * dequantised bf16 weights [gate I*H | up I*H | down H*I] and, if bits<16, the canonical
 * codes/scales/zeros in the same matrix order. */
void or_expert_tier(const uint16_t* master, int32_t H, int32_t I, int32_t g,
                    int32_t high_bits, int32_t low_bits, int32_t tier_high,
                    uint16_t* w_deq, uint8_t* codes, uint16_t* scales, uint8_t* zeros);

/* ---- O-5 MoE FFN (Eq. 1, routed term) ----
 * weights[e] points to the dequantised bf16 weights of expert e at its stable tier.
 * Y[T][k][H] per-(token,rank) outputs, y[T][H]. */
void or_moe_ffn(const uint16_t* x, const int32_t* idx, const float* gate,
                const uint16_t* const* weights, int32_t T, int32_t k, int32_t H, int32_t I,
                uint16_t* Y, uint16_t* y, int32_t nthreads);

/* ---- O-3/O-6 controller + pool ledger state machine (Alg.1 PAPER.md:183-218;
 *      §3.3; §3.4; §3.5) ---- */
typedef struct or_ctrl or_ctrl;
or_ctrl* or_ctrl_create(int32_t E, int32_t n_hot, int32_t n_spare, double alpha, int32_t period,
                        int32_t warmup, int32_t dwell, int32_t lag);
void     or_ctrl_destroy(or_ctrl* c);
void     or_ctrl_fold(or_ctrl* c, const uint64_t* mass, uint64_t B_tot);
/* returns number of commands written (>=0), or -1 when no plan is due at this step.
 * dir: +1 promote, -1 demote, 0 relayout move (finalize only).  *finalize set to 1 at t==W. */
int32_t  or_ctrl_plan(or_ctrl* c, int32_t* expert, int32_t* dir, int32_t* dst, int32_t* finalize);
/* manual command (Alg. 1 EnqueueUpgrade/EnqueueDowngrade for a given expert);
 * returns 0 ok, 1 wrong tier or warm-up not finished, 2 range, 4 pool exhausted (deferred), 5 busy */
int32_t  or_ctrl_command(or_ctrl* c, int32_t e, int32_t dir);
void     or_ctrl_state(const or_ctrl* c, double* S, int32_t* tier, int32_t* slot, uint32_t* version,
                       int64_t* last, int32_t* in_flight, int64_t* t, double* tau,
                       int32_t* used_hi, int32_t* cap_hi, int32_t* used_lo, int32_t* cap_lo);
int32_t  or_ctrl_owner(const or_ctrl* c, int32_t hi, int32_t slot);
void     or_ctrl_debug_set(or_ctrl* c, const double* S, const int32_t* tier, double tau, int64_t t);

/* ---- ledger primitive (SPEC.md:247-265 alloc/free) ---- */
int32_t or_ledger_alloc(int32_t* owner, int32_t cap, int32_t who);   /* lowest free, -1 exhausted */
int32_t or_ledger_free(int32_t* owner, int32_t cap, int32_t slot, int32_t who); /* 0 ok, -1 corrupt */

/* f-1 cross-layer correlation prefetch */
void    or_corr_update(uint32_t* corr, const int32_t* idx_a, const int32_t* idx_b, int32_t T, int32_t k, int32_t E);
int32_t or_prefetch_candidates(const uint32_t* corr, const int32_t* idx, int32_t T, int32_t k, int32_t E,
                               const int32_t* tier, const int32_t* in_flight, const int32_t* hi_owner, int32_t cap_hi,
                               int32_t f, int32_t* out_e, int32_t* out_b);

/* f-3 shared expert (Eq. 1 first sum; DESIGN.md R-S1) */
void or_shared_ffn(const uint16_t* x, const uint16_t* Ws, int32_t T, int32_t H, int32_t I, uint16_t* Ys,
                   int32_t nthreads);
void or_combine_shared(const uint16_t* Ys, const uint16_t* Y, int32_t T, int32_t k, int32_t H, uint16_t* y);

#ifdef __cplusplus
}
#endif
#endif
