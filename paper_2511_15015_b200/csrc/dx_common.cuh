// dx_common.cuh -- shared device/host definitions of the DynaExq B200 library (product code).
// No code here is shared with oracle/ (the CPU oracle is an independent implementation).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/dx.h"

#define DX_WARP 32
#define DX_NUM_SMS 148

typedef unsigned long long u64;
typedef long long i64;

// ---------------------------------------------------------------- slot layout (DESIGN.md R-P1)
// Quantised slot of one expert at `bits`: codes gate[I][H*b/8] | up[I][H*b/8] | down[H][I*b/8]
// | scales (bf16, [rows][K/g]) gate | up | down | zeros (u8) gate | up | down; every sub-array
// 128 B aligned (the three matrices have I*H elements each, so sub-arrays are equal-sized).
// bf16 slot: gate[I][H] | up[I][H] | down[H][I].
struct SlotLayout {
    int bits;
    i64 codes_stride;   // bytes per matrix of codes (or bf16 matrix)
    i64 scales_off, scales_stride;
    i64 zeros_off, zeros_stride;
    i64 bytes;          // padded slot size
};

static inline i64 dx_up(i64 v, i64 a) { return (v + a - 1) / a * a; }

static inline SlotLayout dx_slot_layout(int H, int I, int g, int bits) {
    SlotLayout s{};
    s.bits = bits;
    i64 n = (i64)I * H;
    if (bits == 16) {
        s.codes_stride = n * 2;
        s.scales_off = s.zeros_off = 3 * n * 2;
        s.scales_stride = s.zeros_stride = 0;
        s.bytes = dx_up(3 * n * 2, 1024);
        return s;
    }
    s.codes_stride = dx_up(n * bits / 8, 128);
    s.scales_off = 3 * s.codes_stride;
    s.scales_stride = dx_up(n / g * 2, 128);
    s.zeros_off = s.scales_off + 3 * s.scales_stride;
    s.zeros_stride = dx_up(n / g, 128);
    s.bytes = dx_up(s.zeros_off + 3 * s.zeros_stride, 1024);
    return s;
}

// A matrix view inside a slot: rows x K, at `bits`.
struct MatView {
    const uint8_t* codes;     // packed codes, or bf16 data when bits == 16
    const __nv_bfloat16* scales;
    const uint8_t* zeros;
    int bits;
};

// ---------------------------------------------------------------- controller state (device)
// Arrays indexed [layer * E + e] (owners: [layer * (E + s) + slot]).
struct Ctrl {
    int32_t* tier;         // 1 HIGH, 0 LOW (published / stable)
    int32_t* slot;         // published block index within the tier region
    uint32_t* version;
    double* S;             // EMA hotness (Eq. 2)
    uint32_t* cnt;         // counters accumulated since the last fold (R-H1)
    u64* mass;
    i64* last;             // step of the last transition
    int32_t* pend_dir;     // +1 / -1 in flight, 0 none
    int32_t* pend_dst;
    i64* pend_at;
    int32_t* lo_owner;     // -1 free, else expert
    int32_t* hi_owner;
    i64* t;                // [L] folds done
    double* tau;           // [L]
    int32_t* cap_lo;       // [L]
    int32_t* cap_hi;       // [L]
    int32_t* plan_n;       // [L]
    int4* plan_cmd;        // [L * E] (expert, dir, dst, src)
    u64* tstats;           // [2] promotions, demotions issued (profiling counters)
    int E, s, n_hot, W, Tp, dwell, lag;
    double alpha;
};

#define DX_NEVER (-(i64)(1ULL << 61))

#ifdef __CUDACC__
// a10 + a14 for one layer, run by ONE thread block (any size): Eq. 2 with Alg. 1's passive
// decay, S <- alpha*S + (1-alpha)*gbar in fp64 without contraction (R-H2), counters cleared, then the
// registration of transitions due at the new step (R-T1): table flip, version++, the old block reclaimed
// (PAPER.md:238).  Used by k_fold and by the combine kernel's fold block (fused step).
__device__ __forceinline__ void fold_layer(const Ctrl& c, int layer, u64 B_tot, double oma) {
    const int E = c.E;
    const i64 t_new = c.t[layer] + 1;
    __syncthreads();
    const double denom = __dmul_rn((double)B_tot, 16777216.0);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int i = layer * E + e;
        const double gbar = B_tot ? __ddiv_rn((double)c.mass[i], denom) : 0.0;
        c.S[i] = __dadd_rn(__dmul_rn(c.alpha, c.S[i]), __dmul_rn(oma, gbar));
        c.cnt[i] = 0;
        c.mass[i] = 0;
        if (c.pend_dir[i] != 0 && c.pend_at[i] == t_new) {      // registration + reclaim
            const int old = c.slot[i];
            const int ob = layer * (E + c.s);
            if (c.pend_dir[i] > 0) { c.lo_owner[ob + old] = -1; c.tier[i] = 1; }
            else                   { c.hi_owner[ob + old] = -1; c.tier[i] = 0; }
            c.slot[i] = c.pend_dst[i];
            c.version[i] += 1;
            c.pend_dir[i] = 0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) c.t[layer] = t_new;
}
#endif

// ---------------------------------------------------------------- programmatic dependent launch
// Every hot-path kernel waits for its predecessor's memory with griddepcontrol.wait (a no-op when it
// was launched without the PDL attribute) and immediately allows its successor to be scheduled, so
// launch latency and prologues (barrier init, TMEM alloc, descriptor prefetch) overlap the tail of the
// previous kernel.
#define DX_GRID_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define DX_GRID_LAUNCH() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
static inline cudaError_t dx_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                    bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#endif
extern bool g_dx_pdl;   // library-wide switch (default on; DX_PDL=0 disables)

// Function attributes (large dynamic smem) are per device context: true the first time it is called for
// the current device with this mask (one static mask per kernel).
static inline bool dx_first_on_device(unsigned long long& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

// ---------------------------------------------------------------- numerics
__device__ __forceinline__ float dx_bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

// dx_expf (DESIGN.md R-G2): every step an IEEE-exact op, no contraction; 2^n applied exactly.
__device__ __forceinline__ float dx_expf(float x) {
    if (x < -103.0f) return 0.0f;
    float n = rintf(__fmul_rn(x, 0x1.715476p+0f));
    float r = __fmaf_rn(n, -0x1.62e4p-1f, x);
    r = __fmaf_rn(n, -0x1.7f7d1cp-20f, r);
    float p = 0x1.a01a02p-13f;            // 1/7!
    p = __fmaf_rn(p, r, 0x1.6c16c2p-10f); // 1/6!
    p = __fmaf_rn(p, r, 0x1.111112p-7f);  // 1/5!
    p = __fmaf_rn(p, r, 0x1.555556p-5f);  // 1/4!
    p = __fmaf_rn(p, r, 0x1.555556p-3f);  // 1/3!
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    int ni = (int)n;
    if (ni >= -126) return __fmul_rn(p, __int_as_float((ni + 127) << 23));
    return __fmul_rn(__fmul_rn(p, 0x1p-64f), __int_as_float((ni + 64 + 127) << 23));
}

// ---------------------------------------------------------------- host helpers
struct DxErr;
void dx_set_error(const char* fmt, ...);
#define DX_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess) {                                                             \
            dx_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            return DX_ERR_CUDA;                                                              \
        }                                                                                    \
    } while (0)

// ---------------------------------------------------------------- kernel launchers (per file)
// k_quant.cu
void launch_quantize(const void* src, int src_bits, const uint8_t* src_scales, const uint8_t* src_zeros,
                     int64_t N, int64_t K, int g, int bits, uint8_t* codes, __nv_bfloat16* scales,
                     uint8_t* zeros, cudaStream_t st);
void launch_dequantize(const uint8_t* codes, const __nv_bfloat16* scales, const uint8_t* zeros,
                       int64_t N, int64_t K, int g, int bits, __nv_bfloat16* out, cudaStream_t st);
// quantise all three matrices of a slot image into a slot image of `bits`
void launch_quantize_slot(const uint8_t* src_slot, const SlotLayout& src, uint8_t* dst_slot,
                          const SlotLayout& dst, int H, int I, int g, cudaStream_t st);

// k_route.cu
struct RouteWs {
    float* logits;        // [T][E]
    int32_t* idx;         // [T][k]
    float* gate;          // [T][k]
    int32_t* hist;        // [nblk][E]
    int32_t* base;        // [nblk][E]
    int32_t* off;         // [E+1]
    int32_t* act_e;       // [E] active experts: HIGH tier first, each tier ascending
    int32_t* n_act;       // [1]
    int32_t* perm;        // [T*k] entry (t*k+j) at each permuted row
    int32_t* inv;         // [T*k] permuted row of entry
    u64* stats;           // [4] device counters: weight bytes gate/up, down, active experts, -
    unsigned* done;       // [1] route-block completion counter (last block runs the scan)
    int16_t* ent;         // [T*k] decode routing: expert of every entry (cross-CTA exchange)
    uint32_t* gm;         // [T*k] decode routing: rint(gate * 2^24) of every entry
    unsigned* gbar;       // [2] decode routing: grid barrier {arrivals, generation}
};
struct RouteStats {       // profiling: algorithmic weight bytes per touched expert [tier][phase]
    const int32_t* tier;
    u64 b00, b01, b10, b11;
    u64* stats;
};
int route_blocks(int T);
// logits[t][e] = x[t] . W_r[e] (+ bias[e]), fp32 (tensor-core products, deterministic sum order)
void launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, int T, int E, int H,
                   float* logits, cudaStream_t st);
// tier: layer table (or NULL); bytes[tier][phase]: algorithmic weight bytes of one expert
void launch_route(const float* logits, int T, int E, int k, int e_lo, const RouteWs& ws,
                  uint32_t* cnt_acc, u64* mass_acc, const int32_t* tier, const u64 (&bytes)[2][2], cudaStream_t st);
// decode batches (route_dec_ok): a1-a4 in ONE multi-CTA launch -- router logits (router mode, wr != NULL) or
// the given logits (trace mode), top-k + gates, hotness counters, offsets, active list, stable perm / inv and
// the gather of x rows into Xp -- with two grid-wide barriers between the phases
bool route_dec_ok(int T, int E, int k);
void launch_route_dec(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, const float* logits_in,
                      int T, int E, int k, int H, int e_lo, const RouteWs& ws, uint32_t* cnt_acc, u64* mass_acc,
                      const int32_t* tier, const u64 (&bytes)[2][2], __nv_bfloat16* Xp, cudaStream_t st);
// stable placement of every (t, j) entry; Xp != NULL also gathers x rows in permuted order
// rowmap != NULL: entry i's source row is rowmap[i] (f-2 deduplicated EP rows) instead of i / k
void launch_place(int T, int E, int k, const RouteWs& ws, const __nv_bfloat16* x, int H, __nv_bfloat16* Xp,
                  cudaStream_t st, const int32_t* rowmap = nullptr);
// f-2 deduplicated EP dispatch (source side, after routing + placement over global experts): mark [G][T] scratch,
// triples [G][3] {unique rows, entries, T_src} per owner, send_rows (owner blocks in order), meta [T*k] int4
// {local expert, gate bits, row within the owner block}
void launch_dedup_dispatch(const RouteWs& ws, int T, int k, int E_loc, int G, const __nv_bfloat16* x, int H,
                           int32_t* mark, int32_t* triples, __nv_bfloat16* send_rows, int4* meta, cudaStream_t st);
// owner side: meta4 [R] (source order) -> meta2 {expert, gate} and rowmap (row among the received rows); eoff / roff:
// per-source entry / row offsets, G + 1 values each (G <= 8)
void launch_dedup_fix(const int4* meta4, int R, int G, const int32_t* eoff, const int32_t* roff, int2* meta2,
                      int32_t* rowmap, cudaStream_t st);
// a8 combine; with fold != NULL one extra block also runs the layer's EMA fold + publication (a10, a14)
struct FoldReq {
    int layer;
    u64 B_tot;
};
// shared_base >= 0: row shared_base + t of Y holds token t's shared-expert term, summed first (f-3, R-S1)
void launch_combine(const __nv_bfloat16* Y, int T, int k, int H, __nv_bfloat16* y, cudaStream_t st,
                    const int32_t* inv = nullptr, const Ctrl* ctrl = nullptr, const FoldReq* fold = nullptr,
                    int shared_base = -1);
// f-3: the shared expert's rows (entries T*k .. T*k+T-1: perm, gate 1, Xp = x) appended after the routed ones, the
// shared expert (id E) listed first among the active experts; stats: its bytes added to the profiling counters
void launch_shared_rows(const RouteWs& ws, int T, int k, int E, int H, const __nv_bfloat16* x, __nv_bfloat16* Xp,
                        u64 b0, u64 b1, cudaStream_t st);
// expert parallelism: owner-side routing from received (local expert, gate) rows (k = 1), and the
// source-side dispatch metadata / per-owner counts
void launch_route_given(const int2* meta, int R, int E, const RouteWs& ws, uint32_t* cnt_acc, u64* mass_acc,
                        const int32_t* tier, const u64 (&bytes)[2][2], int32_t* err, cudaStream_t st);
// counts: [G] rows per owner (or NULL); pairs: [G] {rows per owner, T_src} for the NCCL count exchange (or NULL)
void launch_ep_meta(const RouteWs& ws, int n, int E_loc, int G, int2* meta, int32_t* counts, int2* pairs, int T_src,
                    cudaStream_t st);

// ep_nccl.cu: the NCCL transport of expert parallelism (dlopen'd libnccl, host API)
dx_status ep_nccl_available();
int ep_nccl_version();
dx_status ep_nccl_unique_id(void* id128);
dx_status ep_nccl_init(const void* id128, int G, int rank, void** comm);
void ep_nccl_destroy(void* comm);
dx_status ep_nccl_exchange_counts(void* comm, int G, int per, const int32_t* tup, int32_t* recv_tup, cudaStream_t st);
dx_status ep_nccl_exchange_rows(void* comm, int G, int H, const void* send_rows, const int* sc, const int* soff,
                                void* recv_rows, const int* rc, const int* roff, const void* send_meta, const int* se,
                                const int* seoff, void* recv_meta, const int* re, const int* reoff, int mi,
                                cudaStream_t st);
// E: global expert count (range check), e_cnt: local experts counted ([e_lo, e_lo + e_cnt))
void launch_counts_from(const int32_t* idx, const float* gate, int T, int E, int e_cnt, int k, int e_lo,
                        uint32_t* cnt_acc, u64* mass_acc, int32_t* err, cudaStream_t st);

// k_expert.cu
struct ExpertArgs {
    const uint8_t* arena_layer;   // base of the layer region
    const int32_t* tier;          // [E] of this layer
    const int32_t* slot;
    i64 hi_base;                  // byte offset of the HIGH region inside the layer region
    SlotLayout hi, lo;
    int H, I, g, k;
};
void launch_expert_ffn(const ExpertArgs& a, const __nv_bfloat16* x, const float* gate, const RouteWs& ws,
                       int T, int E, __nv_bfloat16* act, __nv_bfloat16* Y, cudaStream_t st, cudaEvent_t mid);

// k_gemm.cu (tcgen05 grouped GEMM)
#include <cuda.h>
struct GemmMaps {
    // A operands.  gate/up maps are 4-D {K, rows, matrix (gate, up), slot}: one box = 64 gate rows + the
    // 64 matching up rows; down maps are 3-D {K, rows, slot}, 128-row boxes.
    CUtensorMap a16_gu, a16_dn;     // bf16 HIGH region, 64-element K boxes, 128 B swizzle
    CUtensorMap ahi_gu, ahi_dn;     // raw codes of a quantised HIGH region, one 64-wide K chunk per box
    CUtensorMap alo_gu, alo_dn;     // raw codes of the LOW region, one 64-wide K chunk per box
    CUtensorMap whi_gu, whi_dn;     // the same, 128 B of codes per row per box (decode stages), 128 B swizzle
    CUtensorMap wlo_gu, wlo_dn;
    // B operands (token rows [rows][K] bf16, 128 B swizzle)
    CUtensorMap xb[4];              // 2-D boxes {64, 16/32/64/128}
    CUtensorMap xw;                 // 2-D box {64, 256}: the wide prefill tiles of k_wide
    CUtensorMap xb192;              // 2-D box {64, 192}: k_gemm's prefill tiles
    CUtensorMap xb1[4], xk1[3];     // fused decode launch: the down phase's B maps (act rows)
    CUtensorMap xk[3];              // 3-D {64, rows, K/64}: boxes {64,16,4}, {64,32,4}, {64,16,8} (decode int stages)
};
struct GemmArgs {
    const uint8_t* layer;
    i64 hi_base;
    SlotLayout hi, lo;
    const int32_t* tier;
    const int32_t* slot;
    const int32_t* off;
    const int32_t* act_e;
    const int32_t* n_act;
    const int32_t* perm;
    const float* gate;
    int H, I, g, k;
    int E_loc, shared_slot;         // f-3: expert id E_loc is the layer's shared expert, HIGH tier, block shared_slot
    __nv_bfloat16* act;
    __nv_bfloat16* Y;
    int* sched;                     // [phase][ticket counter, CTAs done]: dynamic work-item hand-out, zero
                                    // between launches (the last CTA of a launch resets it)
    int skip_bf16;                  // prefill k_gemm: the leading bf16 (HIGH, 16-bit) experts are k_wide's
    int* dn_done;                   // fused decode launch: gate/up items finished per active expert (self-resetting)
    int dbg;                        // performance experiments only (DX_GEMM_DBG): 4 skip the A-in-TMEM MMAs,
                                    // 5 skip the dequant transform, 6 both, 13 = 6 with plain
                                    // arrivals instead of tcgen05.commit on int stages
};
bool gemm_decode_cfg(int T);

void gemm_trap_init();                            // host-mapped watchdog record (once per process)
int gemm_trap_report(char* buf, size_t n);        // appends the record, if a k_gemm wait timed out
void launch_gemm(int phase, bool dec, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st);
// prefill: the bf16 (HIGH) experts' items as 128 x 256 tiles (k_wide); k_gemm then takes only the others (skip_bf16)
void launch_wide(int phase, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st);
bool wide_enabled();

// k_ctrl.cu
void launch_fold(const Ctrl& c, int layer, u64 B_tot, cudaStream_t st);
void launch_plan(const Ctrl& c, int layer, int finalize, cudaStream_t st);
// f-1 cross-layer correlation prefetch (k_ctrl.cu)
void launch_corr(const int32_t* idx_prev, const int32_t* idx, int T, int k, int E, uint32_t* corr, int32_t* idx_save,
                 cudaStream_t st);
void launch_prefetch(const Ctrl& c, int layer, const uint32_t* corr, const int32_t* idx_cur, int T, int k, int f,
                     int4* out, int32_t* n_out, cudaStream_t st);
struct XferArgs {
    uint8_t* layer_base;
    i64 hi_base;
    SlotLayout hi, lo;
    const uint8_t* const* hi_img;   // [E] device-accessible pointers to HIGH images (host-mapped)
    int H, I, g;
};
void launch_transitions(const Ctrl& c, int layer, const XferArgs& x, int max_cmds, int mode,
                        cudaStream_t st);
