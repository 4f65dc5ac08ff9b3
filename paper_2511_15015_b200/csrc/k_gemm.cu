// k_gemm.cu -- tcgen05 grouped expert GEMMs over the slot pool (a6 gate/up + SwiGLU, a7 down + gate
// scaling), one persistent kernel per phase, every touched expert at its stable tier.
//   Eq. 1: E_j(x) = W_down (silu(W_gate x) * W_up x).
//
// Swap-AB: the weights are the M = 128 operand, the tokens of one expert are N (16..128, chosen per
// chunk from the expert's token count), the accumulator D[128 x N] fp32 lives in TMEM (two buffers, so
// the epilogue of one chunk overlaps the MMAs of the next).  Persistent CTAs (one per SM) walk the work
// items (expert, 128-row block) round-robin.
//
// Stage ring (6 x 32 KB smem): an A region (16 KB) and a B region (16 KB).  A bf16 stage holds one
// 64-wide K chunk: A = 128 weight rows TMA'd straight into the 128 B-swizzled UMMA layout.  A quantised
// stage holds KS = 4 (int4) or 8 (int2) K chunks of raw codes (16 KB), so every stage carries 16 KB of
// weight bytes whatever the tier (the HBM stream stays deep), with KS B sub-tiles.  Raw codes are
// dequantised exactly (bf16_rn((q-z)s), R-Q1) by two transform warp groups straight into a ring of
// 32-column TMEM A buffers (lane = weight row) that feeds tcgen05.mma with A in tensor memory.
// Gate/up items take 64 gate rows (A rows 0-63) and the matching 64 up rows (64-127); the SwiGLU pairs
// meet through a small smem exchange in the epilogue.
// Warp roles (480 threads): 0 TMA producer, 1 TMEM owner + MMA issuer, 2-9 transform, 10-13 epilogue,
// 14 scheduler.  Work items are handed out dynamically (one global ticket counter per launch, items in
// the routing kernel's HIGH-tier-first order, so the heavy items go first and the tail is a light one):
// the scheduler warp claims a ticket, decodes it and publishes it through a 2-entry smem ring that every
// other role walks in the same order.
#include "dx_common.cuh"
#include "dx_sm100.cuh"
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <type_traits>

using namespace sm100;

namespace {

#ifndef DX_GEMM_NTW
#define DX_GEMM_NTW 16
#endif
constexpr int NTW = DX_GEMM_NTW;              // dequant transform warps (groups of 4: one per TMEM lane quarter)
constexpr int NG = NTW / 4;                   // transform groups
constexpr int W_EPI = 2 + NTW;                // first epilogue warp
// Epilogue warpgroups ("teams", team t drains accumulator buffer t): one for decode (the dequant warps
// need the registers: 80 at 736 threads), two for prefill (the SwiGLU/scatter epilogue was a limiter:
// measured +4 % prefill TFLOP/s; the same layout costs decode 7-10 % through the 72-register cap).
template <bool DEC>
struct Roles {
    static constexpr int EPI_TEAMS = DEC ? 1 : 2;
    static constexpr int W_SCHED = W_EPI + 4 * EPI_TEAMS;     // scheduler warp
    static constexpr int THREADS = 32 * (W_SCHED + 1);
    static constexpr int N_CONSUMERS = W_SCHED;               // warps that read the item ring
};
constexpr int KCH = 64;                       // K elements per chunk (128 B of bf16 per row)
constexpr int STAGES = 6;
constexpr int A_BYTES = 128 * 128;            // A / raw region per stage
constexpr int B_REGION = 16384;               // B region per stage
constexpr int STAGE_BYTES = A_BYTES + B_REGION;
constexpr int XCH_BYTES = 64 * 32 * 4;        // epilogue SwiGLU exchange: 64 rows x 32 columns fp32
constexpr int TPRE_BYTES = (512 + 1) * 4 + 12;   // prefill: per-active-expert N-tile prefix
constexpr int EMAX = 512;
constexpr int ETAB_BYTES = EMAX * 16;            // decode: {r0, m, slot, tier} per active expert
#ifndef DX_GEMM_RING
#define DX_GEMM_RING 2
#endif
constexpr int RING = DX_GEMM_RING;                       // claimed work items in flight per CTA (small: balance)
constexpr int GTAB = 16;                      // scale/zero groups per row staged in smem per item (G <= 16)
constexpr int TAB_BYTES = 128 * GTAB * 3;     // one item's table: [128 rows][G] bf16 scales, then u8 zeros

// DEC: decode configuration (T <= 64): N <= 64 for bf16, 32 for int4, 16 for int2 with KS chunks per
// quantised stage; otherwise (prefill) N <= 128 and one chunk per stage for every tier.
template <bool DEC>
struct Cfg {
    // prefill: N tiles of 192 tokens (an int item's dequantised chunk feeds 1.5x the MMAs of a 128 tile; the two
    // 192-column accumulators leave 4 TMEM A buffers, one per dequant group), 4 stages of 16 KB A + 24 KB B
    static constexpr int NBMAX = DEC ? 64 : 192;
    static constexpr int STG = DEC ? STAGES : 4;
    static constexpr int SBYTES = DEC ? STAGE_BYTES : A_BYTES + 192 * 128;
    static constexpr int ACH = DEC ? 4 : 1;                    // K chunks per TMEM A buffer (32 columns each)
    static constexpr int NA = (512 - 2 * NBMAX) / (32 * ACH);  // TMEM A buffers: 3 (decode) / 8 (prefill)
    static constexpr int SMEM = 1024 + STG * SBYTES + Roles<DEC>::EPI_TEAMS * XCH_BYTES + 2048 + RING * 32 + 2 * TAB_BYTES +
                                (DEC ? ETAB_BYTES : TPRE_BYTES);
    __device__ static int nb(int bits) { return DEC ? (bits == 16 ? 64 : (bits == 4 ? 32 : 16)) : NBMAX; }
    __device__ static int ks(int bits) { return (DEC && bits != 16) ? 16 / bits : 1; }   // int4: 4, int2: 8
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// (bf16 scale | bf16(128 + z) << 16) of group gi from the slot in global memory (tables too wide for smem)
__device__ __noinline__ uint32_t group_sz_global(const uint16_t* scales, const uint8_t* zeros, int gi) {
    return (uint32_t)scales[gi] | ((0x4300u + zeros[gi]) << 16);
}
__device__ __forceinline__ uint32_t bf2_sub_mul(uint32_t v, uint32_t zz, uint32_t ss) {
    __nv_bfloat162 r = __hmul2(__hsub2(*reinterpret_cast<__nv_bfloat162*>(&v), *reinterpret_cast<__nv_bfloat162*>(&zz)),
                               *reinterpret_cast<__nv_bfloat162*>(&ss));
    return *reinterpret_cast<uint32_t*>(&r);
}

// Exact dequantisation of one 64-element chunk of a row (R-Q1): codes at smem ra0 (and ra1 for the second
// 16 B of int4), pair-interleaved packing (pair j at bits {bits*j, 16 + bits*j} of a 32-bit word), so a
// bf16x2 of (128 + q) is (word >> bits*j) & mask | 0x4300_4300; then (. - (128 + z)) * s, each rounded once.
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t m, uint32_t c) {   // (x & m) | c, one LOP3
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "r"(m), "r"(c));
    return d;
}
__device__ __forceinline__ void dequant_chunk(int bits, uint32_t ra0, uint32_t ra1, const uint32_t (&zz)[2],
                                              const uint32_t (&ss)[2], uint32_t (&wv)[KCH / 2], uint32_t magic) {
    if (bits == 4) {
        uint32_t s0, s1, s2, s3, s4, s5, s6, s7;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "r"(ra0));
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s4), "=r"(s5), "=r"(s6), "=r"(s7) : "r"(ra1));
        const uint32_t src[8] = {s0, s1, s2, s3, s4, s5, s6, s7};
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const uint32_t x = src[b >> 2] >> (4 * (b & 3));
            wv[b] = bf2_sub_mul(and_or(x, 0x000F000Fu, magic), zz[b >> 4], ss[b >> 4]);
        }
    } else {
        uint32_t s0, s1, s2, s3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "r"(ra0));
        const uint32_t src[4] = {s0, s1, s2, s3};
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const uint32_t x = src[b >> 3] >> (2 * (b & 7));
            wv[b] = bf2_sub_mul(and_or(x, 0x00030003u, magic), zz[b >> 4], ss[b >> 4]);
        }
    }
}

// Protocol watchdog: a wait that never completes records which barrier (tag), parity, block and thread in a
// host-mapped word array and traps, so a hang surfaces as a launch error with a readable diagnosis
// (gemm_trap_report) instead of a stuck GPU.
__device__ uint32_t* g_gemm_trap = nullptr;
__device__ uint64_t g_gemm_watchdog_ns = 2000000000ull;   // DX_WATCHDOG_S (ncu's instrumented replays need more)
__device__ __noinline__ void gemm_trap(uint32_t tag, uint32_t parity) {
    uint32_t* r = g_gemm_trap;
    if (r && atomicCAS(r, 0u, 0xDEAD0000u | tag) == 0u) {
        r[1] = parity;
        r[2] = blockIdx.x;
        r[3] = threadIdx.x;
        __threadfence_system();
    }
    __trap();
}
#ifndef DX_STATIC_FIRST
#define DX_STATIC_FIRST 0      // 1: each CTA's first work item is blockIdx.x (measured: slower whenever side-stream transfer blocks share SMs: C2 490 K vs 503 K layer-tok/s, exposed switch 7.1 vs 4.5 %)
#endif
#ifndef DX_EPI_BACK
#define DX_EPI_BACK 256        // backoff (ns) of the epilogue's accumulator wait (MMA's drain wait: half)
#endif
#ifndef DX_TBACK
#define DX_TBACK 0             // backoff (ns) of the dequant warps' own waits
#endif
#ifndef DX_GEMM_SPIN
#define DX_GEMM_SPIN 0
#endif
__device__ __forceinline__ bool gtry(uint32_t a, uint32_t parity) {
    return DX_GEMM_SPIN ? mbar_try_wait(a, parity) : mbar_try_wait_sleep(a, parity);
}
// Slow path of a barrier wait, out of line: polls (the watchdog clock is read once per 256 polls) and
// sleeps backoff_ns between polls.  Waiting warps share their sub-partition's issue slots with the dequant
// warps, so every role except the dequant workers backs off.
__device__ __noinline__ void gwait_slow(uint32_t a, uint32_t parity, uint32_t tag, uint32_t backoff_ns) {
    const uint64_t lim = g_gemm_watchdog_ns;
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
#pragma unroll 1
        for (int i = 0; i < 256; ++i) {
            if (mbar_try_wait(a, parity)) return;
            if (backoff_ns) __nanosleep(backoff_ns);
        }
        if (globaltimer_ns() - t0 > lim) gemm_trap(tag, parity);   // default 2 s: a protocol bug
    }
}
__device__ __forceinline__ void gwait(uint64_t* bar, uint32_t parity, uint32_t tag, uint32_t backoff_ns = 0) {
    const uint32_t a = smem_u32(bar);
    if (gtry(a, parity)) return;
    gwait_slow(a, parity, tag, backoff_ns);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Decoded work item: 128-row block mb of an active expert, its token rows [r0, r0+m), tier / slot / bits.
struct Item {
    int mb, r0, m, ti, slot, bits;
    int ph, ae;            // phase (fused decode launch) and active-expert index of the item
};
// Prefill work items are (expert, N tile of NT token rows, row block): the N tiles of every active expert
// are numbered by the prefix tpre[] (so a hot expert's thousands of rows spread over many SMs instead of
// one CTA walking all of them); decode items are (expert, row block) with all of its rows.
__device__ __forceinline__ int4 decode_tiled(const GemmArgs& a, const int32_t* tpre, int n_act, int item, int nmb,
                                             int NT) {
    const int q = item / nmb;
    int lo = 0, hi = n_act - 1;                        // largest a with tpre[a] <= q
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tpre[mid] <= q) lo = mid; else hi = mid - 1;
    }
    const int e = a.act_e[lo];
    const int r0 = a.off[e] + (q - tpre[lo]) * NT;
    const int m = min(NT, a.off[e + 1] - r0);
    return make_int4(r0, m, e < a.E_loc ? a.slot[e] : a.shared_slot, e < a.E_loc ? a.tier[e] : 1);
}
__device__ __forceinline__ int4 decode_raw(const GemmArgs& a, const int4* etab, int item, int nmb) {   // {r0, m, slot, ti}
    if (item / nmb < EMAX) return etab[item / nmb];
    const int e = a.act_e[item / nmb];
    const int r0 = a.off[e];
    return make_int4(r0, a.off[e + 1] - r0, e < a.E_loc ? a.slot[e] : a.shared_slot, e < a.E_loc ? a.tier[e] : 1);
}
// One published work item of the ring: decoded fields + the ticket (>= n_items: no more work).
struct Tick {
    int4 v;            // {r0, m, slot, tier}
    int item, pad[3];
};

// The ii-th item of this CTA, from the ring (every field warp-uniform: read by lane 0, broadcast).  The
// warp then releases the ring entry.  Returns false after the last item.
__device__ __forceinline__ bool take_item(const GemmArgs& a, const Tick* ring, uint64_t* tkfull, uint64_t* tkempty,
                                          int ii, int n_items, int nmb, Item& it, int n0 = -1, int nmb1 = 1) {
    const int sl = ii % RING;
    gwait(&tkfull[sl], (ii / RING) & 1, 10, 128);
    int4 v = ring[sl].v;
    int item = ring[sl].item;
    v.x = __shfl_sync(0xffffffffu, v.x, 0);
    v.y = __shfl_sync(0xffffffffu, v.y, 0);
    v.z = __shfl_sync(0xffffffffu, v.z, 0);
    v.w = __shfl_sync(0xffffffffu, v.w, 0);
    item = __shfl_sync(0xffffffffu, item, 0);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&tkempty[sl]);
    if (item >= n_items) return false;
    if (n0 >= 0 && item >= n0) {                       // fused decode launch: down items follow the gate/up items
        it.ph = 1;
        it.mb = (item - n0) % nmb1;
        it.ae = (item - n0) / nmb1;
    } else {
        it.ph = 0;
        it.mb = item % nmb;
        it.ae = item / nmb;
    }
    it.r0 = v.x;
    it.m = v.y;
    it.slot = v.z;
    it.ti = v.w;
    it.bits = it.ti ? a.hi.bits : a.lo.bits;
    return true;
}

__device__ __forceinline__ int box_rows(int nvalid) {        // B tile rows: power of two in [16, 128]
    int r = 16;
    while (r < nvalid) r <<= 1;
    return r;
}
__device__ __forceinline__ int box_rows_p(int nvalid) {      // k_gemm prefill: 16 .. 128, then 192
    return nvalid <= 128 ? box_rows(nvalid) : 192;
}

template <int PHASE, bool DEC>
__global__ void __launch_bounds__(Roles<DEC>::THREADS, 1) k_gemm(const __grid_constant__ GemmMaps maps, GemmArgs a) {
    constexpr int EPI_TEAMS = Roles<DEC>::EPI_TEAMS, W_SCHED = Roles<DEC>::W_SCHED, N_CONSUMERS = Roles<DEC>::N_CONSUMERS;
    using C = Cfg<DEC>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sS = smem;                                   // [C::STG][A 16 KB | B 16 KB]
    float* xch = reinterpret_cast<float*>(sS + C::STG * C::SBYTES);            // [32 cols][64 rows]
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + EPI_TEAMS * XCH_BYTES);
    uint64_t* full = bars;                                // [C::STG] TMA landed (A or raw, and B)
    uint64_t* empty = full + C::STG;                      // [C::STG] MMA finished with the stage
    uint64_t* aready = empty + C::STG;                    // [NA] transform wrote TMEM A buffer
    uint64_t* aempty = aready + C::NA;                    // [NA] MMA finished with TMEM A buffer
    uint64_t* tfull = aempty + C::NA;                     // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                         // [2] accumulator drained
    uint64_t* tabfull = tempty + 2;                       // [2] scale/zero table of an item landed
    uint64_t* tabempty = tabfull + 2;                     // [2] transform finished with the table
    uint64_t* tkfull = tabempty + 2;                      // [RING] item published by the scheduler
    uint64_t* tkempty = tkfull + RING;                    // [RING] every consumer warp read the item
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tkempty + RING);
    int32_t* ent_s = reinterpret_cast<int32_t*>(tmem_slot + 4);     // [128] epilogue: entry ids
    float* gate_s = reinterpret_cast<float*>(ent_s + 128);           // [128] epilogue: gates
    Tick* ring = reinterpret_cast<Tick*>(reinterpret_cast<uint8_t*>(bars) + 2048);   // [RING] items
    uint8_t* tabs = reinterpret_cast<uint8_t*>(ring + RING);         // [2][TAB_BYTES]
    int32_t* tpre = reinterpret_cast<int32_t*>(tabs + 2 * TAB_BYTES); // [n_act + 1] prefill N-tile prefix
    int4* etab = reinterpret_cast<int4*>(tabs + 2 * TAB_BYTES);       // decode: [EMAX] the active experts' items

    // PHASE 2 (decode only): ONE launch runs the gate/up items and then the down items of every active expert; a
    // down item is handed out only after all gate/up items of its expert have written their act rows (per-expert
    // completion counters), so the down work of early experts overlaps the gate/up tail of late ones.
    constexpr bool FUSED = PHASE == 2;
    static_assert(!FUSED || DEC, "the fused launch is the decode configuration");
    const int nmb0 = a.I / 64, nmb1 = (a.H + 127) / 128;
    const int nmb = PHASE == 1 ? nmb1 : nmb0;             // (fused: of the first n0 items)
    const int nk_[2] = {a.H / KCH, a.I / KCH};
    const int G_[2] = {a.H / a.g, a.I / a.g};             // quantisation groups per weight row
    const bool tab_ok_[2] = {G_[0] <= GTAB, G_[1] <= GTAB};   // per-item scale/zero tables staged by TMA
    // warp index made provably warp-uniform: role branches are uniform and the single-thread issue paths
    // keep their operands in uniform registers
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;

    // prologue independent of the predecessor kernels (overlaps their tail under PDL)
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STG; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1 + NTW); }
        for (int b = 0; b < C::NA; ++b) { mbar_init(&aready[b], DEC ? NTW : 4); mbar_init(&aempty[b], 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4);
            mbar_init(&tabfull[b], 1); mbar_init(&tabempty[b], NTW);
        }
        for (int b = 0; b < RING; ++b) { mbar_init(&tkfull[b], 1); mbar_init(&tkempty[b], N_CONSUMERS); }
        fence_mbar_init();
        for (int i = 0; i < 4; ++i) tma_prefetch(&maps.xb[i]);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n_act = a.n_act[0];
    int n_items = n_act * nmb;
    const int n0 = FUSED ? n_act * nmb0 : -1;              // fused: items [0, n0) gate/up, [n0, n_items) down
    if (FUSED) n_items = n_act * (nmb0 + nmb1);
    if (!DEC) {
        // N tiles per active expert, exclusive prefix over the active list (n_act <= 512 < blockDim)
        __shared__ int32_t wsum[32];
        const int t = threadIdx.x;
        int v = 0;
        if (t < n_act) {
            const int e = a.act_e[t];
            const bool bf = a.skip_bf16 && (e >= a.E_loc || a.tier[e]);    // k_wide's (bf16 HIGH) expert
            v = bf ? 0 : (a.off[e + 1] - a.off[e] + C::NBMAX - 1) / C::NBMAX;
        }
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        int base = 0;
        for (int w2 = 0; w2 < warp; ++w2) base += wsum[w2];
        if (t <= n_act) tpre[t] = base + x - v;
        __syncthreads();
        n_items = tpre[n_act] * nmb;
    } else {
        // the active experts' rows, slots and tiers, read once into shared memory: the scheduler then
        // decodes a ticket without a dependent chain of global loads per work item
        for (int i = threadIdx.x; i < n_act && i < EMAX; i += Roles<DEC>::THREADS) {
            const int e = a.act_e[i];
            const int r0 = a.off[e];
            etab[i] = make_int4(r0, a.off[e + 1] - r0, e < a.E_loc ? a.slot[e] : a.shared_slot, e < a.E_loc ? a.tier[e] : 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t tmem_a = tmem + 2 * C::NBMAX;          // first TMEM A buffer column

    if (warp == 0) {
        // ------------------------------------------------ TMA producer: the whole warp walks the stages
        // with warp-uniform values (uniform registers, no per-lane serialisation); lane 0 issues
        int st = 0, tc = 0;
        uint32_t ph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w, n0, nmb1); ++ii) {
            const int iph = FUSED ? w.ph : PHASE;
            const int nk = nk_[iph], G = G_[iph];
            const bool tab_ok = tab_ok_[iph];
            const bool qt = w.bits != 16;
            if (FUSED && iph == 1) asm volatile("fence.proxy.async.global;" ::: "memory");   // act rows: generic -> TMA
            if (qt && tab_ok) {
                // this item's scales / zeros: contiguous row spans of the slot's [rows][G] tables
                const int tb = tc & 1;
                gwait(&tabempty[tb], ((tc >> 1) & 1) ^ 1, 1, 128);
                ++tc;
                if (elect_one()) {
                    const SlotLayout& L = w.ti ? a.hi : a.lo;
                    const uint8_t* sb = a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
                    uint8_t* ts = tabs + tb * TAB_BYTES;
                    uint8_t* tz = ts + 128 * GTAB * 2;
                    if (iph == 0) {
                        const uint32_t sbytes = 64 * G * 2, zbytes = 64 * G;
                        mbar_arrive_expect_tx(&tabfull[tb], 2 * (sbytes + zbytes));
                        for (int m = 0; m < 2; ++m) {        // gate rows -> table rows 0-63, up rows -> 64-127
                            const int64_t row = (int64_t)w.mb * 64;
                            bulk_load(ts + m * sbytes, sb + L.scales_off + m * L.scales_stride + row * G * 2, sbytes,
                                      &tabfull[tb]);
                            bulk_load(tz + m * zbytes, sb + L.zeros_off + m * L.zeros_stride + row * G, zbytes,
                                      &tabfull[tb]);
                        }
                    } else {
                        const int rows = min(128, a.H - w.mb * 128);
                        const int64_t row = (int64_t)w.mb * 128;
                        mbar_arrive_expect_tx(&tabfull[tb], rows * G * 3);
                        bulk_load(ts, sb + L.scales_off + 2 * L.scales_stride + row * G * 2, rows * G * 2, &tabfull[tb]);
                        bulk_load(tz, sb + L.zeros_off + 2 * L.zeros_stride + row * G, rows * G, &tabfull[tb]);
                    }
                }
                __syncwarp();
            }
            const CUtensorMap* amap =
                iph == 0 ? (!qt ? &maps.a16_gu : DEC ? (w.ti ? &maps.whi_gu : &maps.wlo_gu) : (w.ti ? &maps.ahi_gu : &maps.alo_gu))
                           : (!qt ? &maps.a16_dn : DEC ? (w.ti ? &maps.whi_dn : &maps.wlo_dn) : (w.ti ? &maps.ahi_dn : &maps.alo_dn));
            const int nb = C::nb(w.bits), ks = C::ks(w.bits);
            const int arow = iph == 0 ? w.mb * 64 : w.mb * 128;
            const CUtensorMap* xbm = (FUSED && iph == 1) ? maps.xb1 : maps.xb;
            const CUtensorMap* xkm = (FUSED && iph == 1) ? maps.xk1 : maps.xk;
            const int kunit = qt ? KCH * w.bits / 8 : KCH;     // A inner coordinate per chunk (bytes / elements)
            for (int c0 = 0; c0 < w.m; c0 += nb) {
                const int rb = DEC ? box_rows(min(nb, w.m - c0)) : box_rows_p(min(nb, w.m - c0));
                const int ri = rb == 16 ? 0 : rb == 32 ? 1 : rb == 64 ? 2 : 3;
                const bool multi = DEC && qt;                   // one B box carries the stage's ks chunks
                const CUtensorMap* bmap = multi ? &xkm[w.bits == 2 ? 2 : ri] : rb == 192 ? &maps.xb192 : &xbm[ri];
                const uint32_t bytes = multi ? A_BYTES + ks * rb * 128 : (qt ? 128 * kunit : A_BYTES) + rb * 128;
                for (int kb0 = 0; kb0 < nk; kb0 += ks) {
                    gwait(&empty[st], ph ^ 1, 2, 128);
                    if (elect_one()) {
                        uint8_t* sA = sS + st * C::SBYTES;
                        mbar_arrive_expect_tx(&full[st], bytes);
                        if (iph == 0) tma_load_4d(sA, amap, &full[st], kb0 * kunit, arow, 0, w.slot);
                        else tma_load_3d(sA, amap, &full[st], kb0 * kunit, arow, w.slot);
                        if (multi) tma_load_3d(sA + A_BYTES, bmap, &full[st], 0, w.r0 + c0, kb0);
                        else tma_load_2d(sA + A_BYTES, bmap, &full[st], kb0 * KCH, w.r0 + c0);
                    }
                    __syncwarp();
                    if (++st == C::STG) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer: warp-uniform walk, lane 0 issues
        // (tcgen05.mma / commit are single-thread instructions; commits must come from the issuing thread)
        int st = 0, ab = 0, cc = 0;
        uint32_t ph = 0, aph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w, n0, nmb1); ++ii) {
            const int nk = nk_[FUSED ? w.ph : PHASE];
            const int nb = C::nb(w.bits), ks = C::ks(w.bits);
            for (int c0 = 0; c0 < w.m; c0 += nb, ++cc) {
                const int rb = DEC ? box_rows(min(nb, w.m - c0)) : box_rows_p(min(nb, w.m - c0));
                const uint32_t idesc = idesc_bf16(128, rb);
                const int buf = cc & 1;
                gwait(&tempty[buf], ((cc >> 1) & 1) ^ 1, 3, DX_EPI_BACK / 2);
                tc_fence_after();
                const uint32_t d = tmem + buf * C::NBMAX;
                for (int kb0 = 0; kb0 < nk; kb0 += ks) {
                    const int kc = min(ks, nk - kb0);
                    gwait(&full[st], ph, 4, 64);
                    tc_fence_after();
                    const uint32_t sA = smem_u32(sS + st * C::SBYTES), sB = sA + A_BYTES;
                    if (w.bits == 16) {
                        const uint64_t da = umma_desc_sw128(sA), db = umma_desc_sw128(sB);
                        if (elect_one()) {
#pragma unroll
                            for (int s = 0; s < KCH / 16; ++s) mma_bf16(d, da + 2 * s, db + 2 * s, idesc, (kb0 | s) != 0);
                        }
                        __syncwarp();
                    } else {
                        const uint64_t db = umma_desc_sw128(sB);
                        const uint32_t bstep = (rb * 128) >> 4;            // B sub-tile stride in descriptor units
                        for (int j0 = 0; j0 < kc; j0 += C::ACH) {         // one TMEM A buffer = ACH chunks
                            gwait(&aready[ab], aph, 5, 64);
                            tc_fence_after();
                            const int jn = min(C::ACH, kc - j0);
                            const uint32_t at = tmem_a + ab * 32 * C::ACH;
                            const uint64_t bj = db + j0 * bstep;
                            const bool first = (kb0 | j0) == 0;
                            if (elect_one()) {
                                if (a.dbg != 4 && a.dbg != 6 && a.dbg != 13) {
                                    if (jn == C::ACH) {
#pragma unroll
                                        for (int q = 0; q < 4 * C::ACH; ++q)
                                            mma_bf16_ts(d, at + 8 * q, bj + (q >> 2) * bstep + 2 * (q & 3), idesc, !first || q);
                                    } else {
                                        for (int j = 0; j < jn; ++j)
#pragma unroll
                                            for (int s = 0; s < 4; ++s)
                                                mma_bf16_ts(d, at + 32 * j + 8 * s, bj + j * bstep + 2 * s, idesc,
                                                            !first || j || s);
                                    }
                                }
                                if (a.dbg == 13) mbar_arrive(&aempty[ab]);   // timing only: no commit latency
                                else mma_commit(&aempty[ab]);
                            }
                            __syncwarp();
                            if (++ab == C::NA) { ab = 0; aph ^= 1; }
                        }
                    }
                    if (elect_one()) {
                        if (a.dbg == 13 && w.bits != 16) mbar_arrive(&empty[st]);
                        else mma_commit(&empty[st]);
                    }
                    __syncwarp();
                    if (++st == C::STG) { st = 0; ph ^= 1; }
                }
                if (elect_one()) mma_commit(&tfull[buf]);
                __syncwarp();
            }
        }
    } else if (warp < W_EPI) {
        // ------------------------------------------------ dequant transform (NTW warps, thread = A row =
        // TMEM lane).  Decode: every TMEM A buffer holds ACH = 4 chunks, group g dequantises chunk(s)
        // ACH/NG*g.. of each; prefill: one chunk per buffer, the NG groups take the buffers in turn.  Every
        // transform warp also releases every stage (empty[] counts 1 MMA commit + NTW warps), so the
        // producer can never lap a warp that is still to observe a stage's phase.
        const int grp = (warp - 2) >> 2;              // 0..NG-1
        const int qa = warp & 3;
        const int r = 32 * qa + lane;
        const uint32_t rsw = r & 7;                        // 128 B swizzle phase of this row
        const uint32_t lane_base = tmem_a + ((uint32_t)(32 * qa) << 16);
        const uint32_t stages_u32 = smem_u32(sS);
        const int gsh = 31 - __clz(a.g);                  // g is a power of two (checked at pool creation)
        uint32_t magic = 0x43004300u;                     // bf16x2 (128, 128): kept in a register for LOP3
        asm volatile("" : "+r"(magic));
        int st = 0, ab = 0, tc = 0, nbuf = 0;
        uint32_t ph = 0, aph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w, n0, nmb1); ++ii) {
            const int iph = FUSED ? w.ph : PHASE;
            const int nk = nk_[iph], G = G_[iph];
            const bool tab_ok = tab_ok_[iph];
            const int mat_rows = iph == 0 ? a.I : a.H;
            if (w.bits == 16) {                           // bf16 stages need no transform: observe their phases
                const int nst = ((w.m + C::nb(16) - 1) / C::nb(16)) * nk;
                for (int s = 0; s < nst; ++s) {
                    gwait(&full[st], ph, 7, 64);         // idle: poll gently
                    __syncwarp();                        // released by every transform warp too, so the
                    if (lane == 0) mbar_arrive(&empty[st]);   // producer can never lap an observer
                    if (++st == C::STG) { st = 0; ph ^= 1; }
                }
                continue;
            }
            // row r of the item's A block: matrix mat (gate 0 / up 1 / down 2), row mrow of it
            const int mat = iph == 0 ? (r >> 6) : 2;
            const int mrow = iph == 0 ? w.mb * 64 + (r & 63) : w.mb * 128 + r;
            const bool valid = mrow < mat_rows;
            const SlotLayout& L = w.ti ? a.hi : a.lo;
            const uint8_t* slot_base =
                a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
            const uint16_t* scales =
                reinterpret_cast<const uint16_t*>(slot_base + L.scales_off + mat * L.scales_stride) + (int64_t)mrow * G;
            const uint8_t* zeros = slot_base + L.zeros_off + mat * L.zeros_stride + (int64_t)mrow * G;
            // scales / zeros: this item's smem table (TMA'd by the producer) when G <= GTAB, else global
            const int tb = tc & 1;
            const uint32_t tsc = smem_u32(tabs + tb * TAB_BYTES) + r * G * 2;             // shared addresses
            const uint32_t tze = smem_u32(tabs + tb * TAB_BYTES + 128 * GTAB * 2) + r * G;
            if (tab_ok) gwait(&tabfull[tb], (tc >> 1) & 1, 6, DX_TBACK);
            // packed (bf16 scale | bf16(128 + z) << 16) of group gi; rows past the matrix: s = 1, z = 0
            auto group_sz = [&](int gi) -> uint32_t {
                if (!valid) return 0x43003f80u;
                return tab_ok ? lds_u16(tsc + 2 * gi) | ((0x4300u + lds_u8(tze + gi)) << 16)
                              : group_sz_global(scales, zeros, gi);
            };
            auto body = [&](auto bits_c) {
                constexpr int BITS = decltype(bits_c)::value;
                constexpr int KS = DEC ? 16 / BITS : 1;     // K chunks per stage
                constexpr int ROWB = KCH * BITS / 8;        // code bytes per row per chunk
                constexpr int NBB = DEC ? (BITS == 4 ? 32 : 16) : C::NBMAX;
                for (int c0 = 0; c0 < w.m; c0 += NBB) {
                    for (int kb0 = 0; kb0 < nk; kb0 += KS) {
                        // every transform thread observes every phase of full[] (no phase aliasing)
                        gwait(&full[st], ph, 7, DX_TBACK);
                        const int cst = st;
                        const uint32_t stage = stages_u32 + st * C::SBYTES;
                        if (++st == C::STG) { st = 0; ph ^= 1; }
                        const int kc = min(KS, nk - kb0);
                        for (int j0 = 0; j0 < kc; j0 += C::ACH, ++nbuf) {
                            const int cab = ab;
                            const uint32_t caph = aph;
                            if (++ab == C::NA) { ab = 0; aph ^= 1; }
                            if (!DEC && (nbuf % NG) != grp) continue;  // prefill: another group's buffer
                            gwait(&aempty[cab], caph ^ 1, 8, DX_TBACK);
                            if (a.dbg != 5 && a.dbg != 6 && a.dbg != 13) {
#pragma unroll
                                for (int h = 0; h < (DEC ? C::ACH / NG : 1); ++h) {
                                    const int jj = DEC ? (C::ACH / NG) * grp + h : 0;   // chunk within the buffer
                                    const int j = j0 + jj;                   // chunk within the stage
                                    if (j < kc) {
                                        const int k0 = (kb0 + j) * KCH;
                                        uint32_t zz[2], ss[2];
                                        const uint32_t v0 = group_sz(k0 >> gsh);
                                        const uint32_t v1 = a.g >= 64 ? v0 : group_sz((k0 + 32) >> gsh);
                                        zz[0] = __byte_perm(v0, 0u, 0x3232);   // bf16(128 + z) in both halves
                                        ss[0] = __byte_perm(v0, 0u, 0x1010);   // bf16 s in both halves
                                        zz[1] = __byte_perm(v1, 0u, 0x3232);
                                        ss[1] = __byte_perm(v1, 0u, 0x1010);
                                        // raw codes of (row r, chunk j): decode stages hold one 128 B-swizzled
                                        // row of KS chunks (16 B unit c of row r at unit c ^ (r & 7)); prefill
                                        // stages one chunk
                                        uint32_t ra0, ra1;
                                        if (DEC) {
                                            const uint32_t row = stage + r * 128;
                                            const uint32_t c = j * ROWB / 16;
                                            ra0 = row + ((c ^ rsw) << 4);
                                            ra1 = row + (((c + 1) ^ rsw) << 4);
                                        } else {
                                            ra0 = stage + r * ROWB;
                                            ra1 = ra0 + 16;
                                        }
                                        uint32_t wv[KCH / 2];      // 32 bf16x2 words = 64 elements
                                        dequant_chunk(BITS, ra0, ra1, zz, ss, wv, magic);
                                        tc_fence_after();
                                        tmem_st32(lane_base + cab * 32 * C::ACH + 32 * jj, wv);
                                    }
                                }
                                tmem_st_wait();
                            }
                            tc_fence_before();
                            __syncwarp();                 // one arrival per warp (arrivals serialise)
                            if (lane == 0) mbar_arrive(&aready[cab]);
                        }
                        __syncwarp();                     // this warp is done reading the stage's codes
                        if (lane == 0) mbar_arrive(&empty[cst]);
                    }
                }
            };
            if (w.bits == 4) body(std::integral_constant<int, 4>{});
            else body(std::integral_constant<int, 2>{});
            if (tab_ok) {                                 // table buffer back to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&tabempty[tb]);
                ++tc;
            }
        }
    } else if (warp == W_SCHED) {
        // ------------------------------------------------ scheduler: claim a ticket, decode it, publish it
        // (the ring is only RING deep, so a CTA never hoards work another SM could start sooner)
        int* ctr = a.sched + (FUSED ? 8 : 2 * PHASE);
        for (int ii = 0;; ++ii) {
            const int sl = ii % RING;
            gwait(&tkempty[sl], ((ii / RING) & 1) ^ 1, 11, 256);
            int item = 0;
            if (lane == 0) {
                item = (DX_STATIC_FIRST && ii == 0) ? (int)blockIdx.x : (DX_STATIC_FIRST ? (int)gridDim.x : 0) + atomicAdd(ctr, 1);   // first item static: no atomic round trip
                if (FUSED && item >= n0 && item < n_items) {
                    // a down item: wait until every gate/up item of its expert has published its act rows
                    const unsigned* dd = reinterpret_cast<const unsigned*>(a.dn_done) + (item - n0) / nmb1;
                    const long long t0 = clock64();
                    while ((int)ld_acquire_u32(dd) < nmb0)
                        if (clock64() - t0 > 8000000000ll) gemm_trap(12, 0);
                }
                ring[sl].v = item >= n_items ? make_int4(0, 0, 0, 0)
                           : DEC ? (FUSED && item >= n0 ? decode_raw(a, etab, item - n0, nmb1) : decode_raw(a, etab, item, nmb))
                                 : decode_tiled(a, tpre, n_act, item, nmb, C::NBMAX);
                ring[sl].item = item;
                mbar_arrive(&tkfull[sl]);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= n_items) break;
        }
    } else {
        // ------------------------------------------------ epilogue: EPI_TEAMS warpgroups of 128 threads; team t
        // drains the chunks that land in accumulator buffer t (cc % 2 == t with two teams), so one team's
        // SwiGLU / scatter overlaps the next chunk's drain by the other.  Each team has its own named
        // barrier and exchange buffer (phase 1 keeps its entry ids / gates in that buffer).
        const int team = (warp - W_EPI) >> 2;
        const int q = warp & 3;                         // TMEM lane quarter this warp may access
        const int et = threadIdx.x - 32 * (W_EPI + 4 * team);   // 0..127
        const uint32_t nbar = 1 + team;
        float* xch_t = xch + team * (XCH_BYTES / 4);
        // phase 1: the chunk's entry ids / gates (decode: <= 64 in the barrier block; prefill: <= 192 in the team's
        // exchange buffer, which phase 1 does not otherwise use)
        int32_t* ent_t = DEC ? ent_s : reinterpret_cast<int32_t*>(xch_t);
        float* gate_t = DEC ? gate_s : xch_t + 256;
        int cc = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w, n0, nmb1); ++ii) {
            const int iph = FUSED ? w.ph : PHASE;
            const int nb = C::nb(w.bits);
            for (int c0 = 0; c0 < w.m; c0 += nb, ++cc) {
                const int buf = cc & 1;
                if (EPI_TEAMS == 2 && buf != team) continue;   // the other team's chunk
                const int nvalid = min(nb, w.m - c0);
                if (iph == 1) {                         // entry ids and gates of this chunk's tokens -> smem
                    for (int i = et; i < nvalid; i += 128) {
                        const int ent = a.perm[w.r0 + c0 + i];
                        ent_t[i] = ent;
                        gate_t[i] = a.gate[ent];
                    }
                }
                gwait(&tfull[buf], (cc >> 1) & 1, 9, DX_EPI_BACK);
                tc_fence_after();
                named_bar(nbar, 128);
                for (int col = 0; col < (a.dbg == 8 ? 0 : nvalid); col += 32) {   // DX_GEMM_DBG=8: skip the epilogue math (timing only)
                    uint32_t v[32];
                    tmem_ld32(tmem + buf * C::NBMAX + ((uint32_t)(32 * q) << 16) + col, v);
                    tmem_ld_wait();
                    if (iph == 0) {
                        // gate rows 0-63 (warps q < 2) meet their up rows 64-127 (q >= 2) through smem, and all
                        // four warps share the SwiGLU: the gate warps take token columns 0-15 of the block (up
                        // values from smem), the up warps columns 16-31 (gate values from smem).
                        // act = bf16(silu(g) * u), silu(g) = g / (1 + e^-g)
                        float* xu = xch_t;                         // [16 cols][64 rows] up values, cols 0-15
                        float* xg = xch_t + 16 * 64;               // [16 cols][64 rows] gate values, cols 16-31
                        const int rr = 32 * (q & 1) + lane;      // row within the 64-row gate/up pair block
                        if (q >= 2) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) xu[j * 64 + rr] = __uint_as_float(v[j]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j) xg[j * 64 + rr] = __uint_as_float(v[16 + j]);
                        }
                        named_bar(nbar, 128);
                        const int f = w.mb * 64 + rr;
                        const int j0 = q < 2 ? 0 : 16;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {        // fully unrolled: v[] stays in registers
                            const int j = j0 + jj;
                            if (col + j < nvalid) {
                                const float gv = q < 2 ? __uint_as_float(v[jj]) : xg[jj * 64 + rr];
                                const float uv = q < 2 ? xu[jj * 64 + rr] : __uint_as_float(v[16 + jj]);
                                const float sg = __fdividef(gv, 1.0f + __expf(-gv));
                                a.act[(size_t)(w.r0 + c0 + col + j) * a.I + f] = __float2bfloat16_rn(sg * uv);
                            }
                        }
                        named_bar(nbar, 128);
                    } else {
                        const int h = w.mb * 128 + 32 * q + lane;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {           // fully unrolled: v[] stays in registers
                            if (col + j < nvalid && h < a.H) {
                                const int ent = ent_t[col + j];
                                a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(gate_t[col + j] * __uint_as_float(v[j]));
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
                named_bar(nbar, 128);                      // ent_s / gate_s / xch reused by the next chunk
            }
            if (FUSED && iph == 0) {                        // this gate/up item's act rows are written: count it
                __threadfence();
                named_bar(nbar, 128);
                if (et == 0) {
                    __threadfence();
                    atomicAdd(a.dn_done + w.ae, 1);
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (threadIdx.x == 0) {                           // the last CTA out resets the ticket counter for the
        int* ctr = a.sched + (FUSED ? 8 : 2 * PHASE);  // next launch (which reads it only after griddepcontrol.wait)
        __threadfence();
        if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(ctr, 0);
            atomicExch(ctr + 1, 0);
            if (FUSED)
                for (int i = 0; i < n_act; ++i) a.dn_done[i] = 0;   // every item is done: counters back to zero
        }
    }
}

// ==========================================================================================================
// k_wide: prefill items of the bf16 (HIGH tier) experts as 128 x 256 tiles (weights M = 128, tokens N <= 256).
// A 128 x 128 tile reads 32 KB of operands per 64-wide K chunk for 2.1 MFLOP; a 128 x 256 tile reads 48 KB for
// 4.2 MFLOP, so the operand stream from L2 per flop drops by a quarter and the tensor pipe issues twice the work
// per barrier round trip.  No dequant warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2-9 two
// epilogue teams (team t drains accumulator buffer t: two 256-column fp32 accumulators = all of TMEM), warp 10
// the scheduler (work items (expert, 256-token tile, row block) over the HIGH experts, through the same global
// ticket counter protocol as k_gemm).  The epilogues are k_gemm's (SwiGLU pairing of gate/up rows; gate scaling
// and the scatter to Y for down).
constexpr int WD_STAGES = 4, WD_B = 256 * 128, WD_STAGE = A_BYTES + WD_B;
constexpr int WD_W_EPI = 2, WD_TEAMS = 2, WD_W_SCHED = WD_W_EPI + 4 * WD_TEAMS, WD_THREADS = 32 * (WD_W_SCHED + 1);
constexpr int WD_SMEM = 1024 + WD_STAGES * WD_STAGE + WD_TEAMS * XCH_BYTES + 1024 + RING * 32 + TPRE_BYTES;
static_assert(WD_SMEM + 2 * 256 * 8 + 128 <= 232448, "k_wide shared memory");

template <int PHASE>
__global__ void __launch_bounds__(WD_THREADS, 1) k_wide(const __grid_constant__ GemmMaps maps, GemmArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sS = smem;
    float* xch = reinterpret_cast<float*>(sS + WD_STAGES * WD_STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + WD_TEAMS * XCH_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = full + WD_STAGES;
    uint64_t* tfull = empty + WD_STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* tkfull = tempty + 2;
    uint64_t* tkempty = tkfull + RING;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tkempty + RING);
    Tick* ring = reinterpret_cast<Tick*>(reinterpret_cast<uint8_t*>(bars) + 1024);
    int32_t* tpre = reinterpret_cast<int32_t*>(ring + RING);
    constexpr int NT = 256;

    const int K = PHASE == 0 ? a.H : a.I;
    const int nmb = PHASE == 0 ? a.I / 64 : (a.H + 127) / 128;
    const int nk = K / KCH;
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < WD_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
        for (int b = 0; b < RING; ++b) { mbar_init(&tkfull[b], 1); mbar_init(&tkempty[b], WD_W_SCHED); }
        fence_mbar_init();
        tma_prefetch(&maps.xw);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n_act = a.n_act[0];
    {
        // 256-token tiles of the HIGH (bf16) experts, exclusive prefix over the active list (n_act <= 513)
        __shared__ int32_t wsum[32];
        int tot = 0;
        for (int base0 = 0; base0 <= n_act; base0 += WD_THREADS) {
            const int t = base0 + threadIdx.x;
            int v = 0;
            if (t < n_act) {
                const int e = a.act_e[t];
                v = (e >= a.E_loc || a.tier[e]) ? (a.off[e + 1] - a.off[e] + NT - 1) / NT : 0;
            }
            int x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            int base = tot;
            for (int w2 = 0; w2 < warp; ++w2) base += wsum[w2];
            if (t <= n_act) tpre[t] = base + x - v;
            int all = 0;
            for (int w2 = 0; w2 < WD_THREADS / 32; ++w2) all += wsum[w2];
            __syncthreads();
            tot += all;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int n_items = tpre[n_act] * nmb;
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    if (warp == 0) {
        int st = 0;
        uint32_t ph = 0;
        Item w;
        const CUtensorMap* amap = PHASE == 0 ? &maps.a16_gu : &maps.a16_dn;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w); ++ii) {
            const int rb = box_rows(w.m);
            const CUtensorMap* bmap = rb == 256 ? &maps.xw : &maps.xb[rb == 16 ? 0 : rb == 32 ? 1 : rb == 64 ? 2 : 3];
            const int arow = PHASE == 0 ? w.mb * 64 : w.mb * 128;
            for (int kb = 0; kb < nk; ++kb) {
                gwait(&empty[st], ph ^ 1, 2, 128);
                if (elect_one()) {
                    uint8_t* sA = sS + st * WD_STAGE;
                    mbar_arrive_expect_tx(&full[st], A_BYTES + rb * 128);
                    if (PHASE == 0) tma_load_4d(sA, amap, &full[st], kb * KCH, arow, 0, w.slot);
                    else tma_load_3d(sA, amap, &full[st], kb * KCH, arow, w.slot);
                    tma_load_2d(sA + A_BYTES, bmap, &full[st], kb * KCH, w.r0);
                }
                __syncwarp();
                if (++st == WD_STAGES) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        int st = 0, cc = 0;
        uint32_t ph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w); ++ii, ++cc) {
            const int rb = box_rows(w.m);
            const uint32_t idesc = idesc_bf16(128, rb);
            const int buf = cc & 1;
            gwait(&tempty[buf], ((cc >> 1) & 1) ^ 1, 3, DX_EPI_BACK / 2);
            tc_fence_after();
            const uint32_t d = tmem + buf * 256;
            for (int kb = 0; kb < nk; ++kb) {
                gwait(&full[st], ph, 4, 64);
                tc_fence_after();
                const uint32_t sA = smem_u32(sS + st * WD_STAGE);
                const uint64_t da = umma_desc_sw128(sA), db = umma_desc_sw128(sA + A_BYTES);
                if (elect_one()) {
#pragma unroll
                    for (int s = 0; s < KCH / 16; ++s) mma_bf16(d, da + 2 * s, db + 2 * s, idesc, (kb | s) != 0);
                    mma_commit(&empty[st]);
                }
                __syncwarp();
                if (++st == WD_STAGES) { st = 0; ph ^= 1; }
            }
            if (elect_one()) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp == WD_W_SCHED) {
        int* ctr = a.sched + 4 + 2 * PHASE;
        for (int ii = 0;; ++ii) {
            const int sl = ii % RING;
            gwait(&tkempty[sl], ((ii / RING) & 1) ^ 1, 11, 256);
            int item = 0;
            if (lane == 0) {
                item = (DX_STATIC_FIRST && ii == 0) ? (int)blockIdx.x : (DX_STATIC_FIRST ? (int)gridDim.x : 0) + atomicAdd(ctr, 1);   // first item static: no atomic round trip
                ring[sl].v = item >= n_items ? make_int4(0, 0, 0, 0) : decode_tiled(a, tpre, n_act, item, nmb, NT);
                ring[sl].item = item;
                mbar_arrive(&tkfull[sl]);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= n_items) break;
        }
    } else {
        // epilogue teams (as k_gemm's prefill epilogue)
        const int team = (warp - WD_W_EPI) >> 2;
        const int q = warp & 3;
        const int et = threadIdx.x - 32 * (WD_W_EPI + 4 * team);
        const uint32_t nbar = 1 + team;
        float* xch_t = xch + team * (XCH_BYTES / 4);
        __shared__ int32_t ent_w[2][256];                 // phase 1: the chunk's entry ids / gates, per team
        __shared__ float gate_w[2][256];
        int32_t* ent_t = ent_w[team];
        float* gate_t = gate_w[team];
        int cc = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, w); ++ii, ++cc) {
            const int buf = cc & 1;
            if (buf != team) continue;
            const int nvalid = w.m;
            if (PHASE == 1) {
                for (int i = et; i < nvalid; i += 128) {
                    const int ent = a.perm[w.r0 + i];
                    ent_t[i] = ent;
                    gate_t[i] = a.gate[ent];
                }
            }
            gwait(&tfull[buf], (cc >> 1) & 1, 9, DX_EPI_BACK);
            tc_fence_after();
            named_bar(nbar, 128);
            for (int col = 0; col < nvalid; col += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + buf * 256 + ((uint32_t)(32 * q) << 16) + col, v);
                tmem_ld_wait();
                if (PHASE == 0) {
                    float* xu = xch_t;
                    float* xg = xch_t + 16 * 64;
                    const int rr = 32 * (q & 1) + lane;
                    if (q >= 2) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) xu[j * 64 + rr] = __uint_as_float(v[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) xg[j * 64 + rr] = __uint_as_float(v[16 + j]);
                    }
                    named_bar(nbar, 128);
                    const int f = w.mb * 64 + rr;
                    const int j0 = q < 2 ? 0 : 16;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int j = j0 + jj;
                        if (col + j < nvalid) {
                            const float gv = q < 2 ? __uint_as_float(v[jj]) : xg[jj * 64 + rr];
                            const float uv = q < 2 ? xu[jj * 64 + rr] : __uint_as_float(v[16 + jj]);
                            const float sg = __fdividef(gv, 1.0f + __expf(-gv));
                            a.act[(size_t)(w.r0 + col + j) * a.I + f] = __float2bfloat16_rn(sg * uv);
                        }
                    }
                    named_bar(nbar, 128);
                } else {
                    const int h = w.mb * 128 + 32 * q + lane;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (col + j < nvalid && h < a.H) {
                            const int ent = ent_t[col + j];
                            a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(gate_t[col + j] * __uint_as_float(v[j]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            named_bar(nbar, 128);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (threadIdx.x == 0) {
        int* ctr = a.sched + 4 + 2 * PHASE;
        __threadfence();
        if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(ctr, 0);
            atomicExch(ctr + 1, 0);
        }
    }
}

template <int PHASE>
void launch_wide_one(const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    static unsigned long long attr_mask = 0;
    if (dx_first_on_device(attr_mask)) cudaFuncSetAttribute(k_wide<PHASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, WD_SMEM);
    const int grid = items < DX_NUM_SMS ? items : DX_NUM_SMS;
    dx_launch(k_wide<PHASE>, dim3(grid), dim3(WD_THREADS), WD_SMEM, st, g_dx_pdl, maps, a);
}

template <int PHASE, bool DEC>
void launch_one(const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    using C = Cfg<DEC>;
    static unsigned long long attr_mask = 0;
    if (dx_first_on_device(attr_mask)) {
        cudaFuncSetAttribute(k_gemm<PHASE, DEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    }
    const int grid = items < DX_NUM_SMS ? items : DX_NUM_SMS;    // persistent: one CTA per SM
    dx_launch(k_gemm<PHASE, DEC>, dim3(grid), dim3(Roles<DEC>::THREADS), C::SMEM, st, g_dx_pdl, maps, a);
}

}  // namespace

bool gemm_decode_cfg(int T) { return T <= 64; }

bool wide_enabled() {
    // opt-in (DX_WIDE=1): with k_gemm's 192-token prefill tiles the single launch is faster (C3 602 vs 571 TFLOP/s)
    static const bool on = [] { const char* e = getenv("DX_WIDE"); return e && atoi(e) != 0; }();
    return on;
}
void launch_wide(int phase, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 0) launch_wide_one<0>(maps, a, max_items, st);
    else launch_wide_one<1>(maps, a, max_items, st);
}

static uint32_t* g_trap_host = nullptr;
void gemm_trap_init() {
    if (g_trap_host) return;
    if (cudaHostAlloc(reinterpret_cast<void**>(&g_trap_host), 64, cudaHostAllocMapped) != cudaSuccess) {
        g_trap_host = nullptr;
        return;
    }
    memset(g_trap_host, 0, 64);
    uint32_t* dptr = nullptr;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), g_trap_host, 0);
    cudaMemcpyToSymbol(g_gemm_trap, &dptr, sizeof(dptr));
    if (const char* w = getenv("DX_WATCHDOG_S")) {
        const uint64_t ns = (uint64_t)(atof(w) * 1e9);
        if (ns > 0) cudaMemcpyToSymbol(g_gemm_watchdog_ns, &ns, sizeof(ns));
    }
}
static const char* const k_trap_names[] = {"?", "tabempty (producer)", "empty (producer)", "tempty (MMA)", "full (MMA)",
                                           "aready (MMA)", "tabfull (transform)", "full (transform)",
                                           "aempty (transform)", "tfull (epilogue)", "tkfull (item ring)",
                                           "tkempty (scheduler)", "gate/up completion (fused scheduler)"};
int gemm_trap_report(char* buf, size_t n) {
    if (!g_trap_host || (g_trap_host[0] >> 16) != 0xDEADu) return 0;
    const uint32_t tag = g_trap_host[0] & 0xFFFFu;
    return snprintf(buf, n, " [k_gemm watchdog: wait on %s, parity %u, block %u, thread %u]",
                    tag < 13 ? k_trap_names[tag] : "?", g_trap_host[1], g_trap_host[2], g_trap_host[3]);
}

void launch_gemm(int phase, bool dec, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 2) {                                  // fused decode FFN (gate/up then down, one launch)
        launch_one<2, true>(maps, a, max_items, st);
        return;
    }
    if (phase == 0) {
        if (dec) launch_one<0, true>(maps, a, max_items, st);
        else launch_one<0, false>(maps, a, max_items, st);
    } else {
        if (dec) launch_one<1, true>(maps, a, max_items, st);
        else launch_one<1, false>(maps, a, max_items, st);
    }
}
