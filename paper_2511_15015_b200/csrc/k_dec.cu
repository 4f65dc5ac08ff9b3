// k_dec.cu -- the decode configuration (T <= 64 tokens per forward) of the grouped expert GEMMs over the
// slot pool: a6 gate/up + SwiGLU and a7 down + gate scaling, one persistent warp-specialised tcgen05 kernel
// per phase, every touched expert read once at its stable tier (Eq. 1 PAPER.md:130:
// E_j(x) = W_down (silu(W_gate x) * W_up x)).
//
// Swap-AB: the weights are the M = 128 operand, an expert's m <= 64 token rows are N (16 / 32 / 64), so every
// work item (expert, 128-row block) is ONE accumulator chunk and every weight tile is read and dequantised
// exactly once.  Stage ring: 6 x (16 KB A | 16 KB B).
//  - bf16 items: a stage is one 64-wide K chunk of 128 weight rows (TMA, 128 B swizzle), SS MMAs.
//  - int items: a stage carries KS K chunks of raw codes (KS = min(16 / bits, 128 / N): 16 KB of codes per
//    stage for N <= 32, the B sub-tiles of those chunks in the B region); code boxes are 128 / 64 / 32 B per
//    row with the matching TMA swizzle.  Four transform groups of four warps (thread = weight row = TMEM
//    lane) dequantise the chunks round-robin, exactly as R-Q1 (bf16_rn((q - z) s)), into a ring of 12
//    32-column TMEM A buffers; the MMAs take A from tensor memory (TS form).
// Barriers: stage full (bf16 TMA), stage empty (one MMA commit: for int stages it follows the MMAs of every
// chunk, which follow the transform's aready, so the codes are no longer read), aready / aempty per TMEM A
// buffer (4 warp arrivals / 1 commit), accumulator full / empty.  The transform warps never touch bf16 items,
// so int stages land on their own barriers, numbered by int-stage sequence (qfull), and each is re-armed only
// after all 16 transform warps have released its previous use (qdone): a warp that skipped a run of bf16
// stages can never mistake an old phase for the one it waits for.  A warp issues a chunk's tcgen05.st and
// signals it (aready) only after the next chunk's arithmetic, so the store latency overlaps work.  Every
// wait re-polls mbarrier.try_wait (each probe blocks in hardware for a short, system-defined time),
// bounded by a watchdog that traps with a readable diagnosis instead of hanging.
// Warp roles (736 threads): 0 TMA producer, 1 TMEM owner + MMA issuer, 2-17 dequant, 18-21 epilogue,
// 22 scheduler (dynamic work items through a global ticket counter; the routing kernel lists HIGH-tier
// experts first, so heavy items go first and the tail is light).
#include "dx_common.cuh"
#include "dx_sm100.cuh"
#include <cstdio>
#include <cstring>
#include <type_traits>

using namespace sm100;

namespace {

constexpr int KCH = 64;                        // K elements per chunk
constexpr int STAGES = 6;
constexpr int A_BYTES = 16384, B_BYTES = 16384, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NTW = 16, NG = 4;                // dequant warps, groups of 4 (one per TMEM lane quarter)
constexpr int ACC_COLS = 64;                   // N <= 64
constexpr int NA = (512 - 2 * ACC_COLS) / 32;  // 12 TMEM A chunk buffers
constexpr int W_EPI = 2 + NTW, W_SCHED = W_EPI + 4;
constexpr int THREADS = 32 * (W_SCHED + 1);
constexpr int N_CONSUMERS = W_SCHED;           // warps that read the item ring
#ifndef DX_DEC_RING
#define DX_DEC_RING 2
#endif
constexpr int RING = DX_DEC_RING;              // work items published ahead of the slowest role (a CTA holding
                                               // more unstarted items than that unbalances the launch's tail)
constexpr int EMAX = 512;                      // active experts held in the shared item table
constexpr int GTAB = 16;
constexpr int TAB_BYTES = 128 * GTAB * 3;
constexpr int XCH_BYTES = 64 * 32 * 4;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + XCH_BYTES + 2 * TAB_BYTES + EMAX * 16 + 2048;

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
__device__ __forceinline__ void lds128(uint32_t a, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
}
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t m, uint32_t c) {   // (x & m) | c, one LOP3
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "r"(m), "r"(c));
    return d;
}
// exact dequant of one bf16x2 pair (R-Q1): ((128 + q) - (128 + z)) is exact, times s rounded once
__device__ __forceinline__ uint32_t deq2(uint32_t q128, uint32_t zz, uint32_t ss) {
    uint32_t d;
    asm("{\n.reg .b32 t;\nsub.rn.bf16x2 t, %1, %2;\nmul.rn.bf16x2 %0, t, %3;\n}" : "=r"(d) : "r"(q128), "r"(zz), "r"(ss));
    return d;
}

// ------------------------------------------------------------------ waits (suspend, watchdog)
__device__ uint32_t* g_dec_trap = nullptr;
__device__ uint64_t g_dec_watchdog_ns = 2000000000ull;
__device__ __noinline__ void dec_trap(uint32_t tag, uint32_t parity) {
    uint32_t* r = g_dec_trap;
    if (r && atomicCAS(r, 0u, 0xDEAD0000u | tag) == 0u) {
        r[1] = parity;
        r[2] = blockIdx.x;
        r[3] = threadIdx.x;
        __threadfence_system();
    }
    __trap();
}
// DX_DEC_BACKOFF=ns: roles other than the dequant warps sleep between polls (their polling loops otherwise
// take issue slots and fma-pipe cycles -- IMAD moves -- from the dequant warps of their sub-partition)
__device__ int g_dec_backoff_ns = 0;
__device__ __noinline__ void dwait_slow(uint32_t a, uint32_t parity, uint32_t tag, int hint) {
    const uint64_t t0 = globaltimer_ns();
    const uint64_t lim = g_dec_watchdog_ns;
    const int back = (tag == 6 || tag == 7 || tag == 8) ? 0 : g_dec_backoff_ns;
    for (;;) {
#pragma unroll 1
        for (int i = 0; i < 64; ++i) {
            if (hint ? mbar_try_wait_sleep(a, parity) : mbar_try_wait(a, parity)) return;
            if (back) __nanosleep(back);
        }
        if (globaltimer_ns() - t0 > lim) dec_trap(tag, parity);
    }
}
// g_dec_wait_hint (DX_DEC_WAIT=1): waits suspend with a time hint instead of re-polling try_wait
__device__ int g_dec_wait_hint = 0;
__device__ __forceinline__ void dwait(uint64_t* bar, uint32_t parity, uint32_t tag) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
    dwait_slow(a, parity, tag, g_dec_wait_hint);
}

// ------------------------------------------------------------------ timeline trace (DX_GEMM_DBG=9, timing study)
constexpr int TR_ITEMS = 32;
__device__ unsigned long long g_dec_trace[2][148][TR_ITEMS][8];
__device__ __forceinline__ void trace(int ph, int ii, int f, unsigned long long v) {
    if (ii < TR_ITEMS && blockIdx.x < 148) g_dec_trace[ph][blockIdx.x][ii][f] = v;
}

// ------------------------------------------------------------------ work items
struct Tick {
    int4 v;            // {r0, m, slot, tier}
    int item, pad[3];
};
struct Item {
    int mb, r0, m, ti, slot, bits;
    int rb, rbi, ks, ksi, wi, nst;   // N box rows (+ index), K chunks per stage (+ index), code box width index, stages
};
__device__ __forceinline__ int box_rows(int m) { return m <= 16 ? 16 : (m <= 32 ? 32 : 64); }
__device__ __forceinline__ void plan_item(Item& it, int nk) {
    it.rb = box_rows(it.m);
    it.rbi = it.rb == 16 ? 0 : (it.rb == 32 ? 1 : 2);
    if (it.bits == 16) {
        it.ks = 1;
        it.ksi = 0;
        it.wi = 0;
        it.nst = nk;
    } else {
        const int kmax = 16 / it.bits, kb = 128 / it.rb;
        it.ks = kmax < kb ? kmax : kb;                       // 2, 4 or 8
        it.ksi = it.ks == 2 ? 1 : (it.ks == 4 ? 2 : 3);
        const int w = it.ks * 8 * it.bits;                   // code bytes per row per stage: 128 / 64 / 32
        it.wi = w == 128 ? 0 : (w == 64 ? 1 : 2);
        it.nst = (nk + it.ks - 1) / it.ks;
    }
}
__device__ __forceinline__ bool take_item(const DecArgs& a, const Tick* ring, uint64_t* tkfull, uint64_t* tkempty,
                                          int ii, int n_items, int nmb, int nk, Item& it) {
    const int sl = ii % RING;
    dwait(&tkfull[sl], (ii / RING) & 1, 10);
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
    it.mb = item % nmb;
    it.r0 = v.x;
    it.m = v.y;
    it.slot = v.z;
    it.ti = v.w;
    it.bits = it.ti ? a.hi.bits : a.lo.bits;
    plan_item(it, nk);
    return true;
}

// swizzled shared address of 16-byte unit c of row r in a code box of 128 / 64 / 32 B per row (TMA
// SWIZZLE_128B / 64B / 32B: unit bits XOR the row bits above the 128-byte line)
__device__ __forceinline__ uint32_t code_unit(uint32_t stage, int r, int c, int wi) {
    if (wi == 0) return stage + r * 128 + ((c ^ (r & 7)) << 4);
    if (wi == 1) return stage + r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
    return stage + r * 32 + ((c ^ ((r >> 2) & 1)) << 4);
}

template <int PHASE>
__global__ void __launch_bounds__(THREADS, 1) k_dec(const __grid_constant__ DecPhaseMaps mp, const DecArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sS = smem;                                                   // [STAGES][A | B]
    float* xch = reinterpret_cast<float*>(sS + STAGES * STAGE_BYTES);     // epilogue SwiGLU exchange
    uint8_t* tabs = reinterpret_cast<uint8_t*>(xch) + XCH_BYTES;          // [2][TAB_BYTES]
    int4* etab = reinterpret_cast<int4*>(tabs + 2 * TAB_BYTES);          // [EMAX] {r0, m, slot, tier} per active expert
    uint64_t* bars = reinterpret_cast<uint64_t*>(etab + EMAX);
    uint64_t* full = bars;                        // [STAGES]
    uint64_t* empty = full + STAGES;              // [STAGES]
    uint64_t* aready = empty + STAGES;            // [NA]
    uint64_t* aempty = aready + NA;               // [NA]
    uint64_t* tfull = aempty + NA;                // [2]
    uint64_t* tempty = tfull + 2;                 // [2]
    uint64_t* tabfull = tempty + 2;               // [2]
    uint64_t* tabempty = tabfull + 2;             // [2]
    uint64_t* tkfull = tabempty + 2;              // [RING]
    uint64_t* tkempty = tkfull + RING;            // [RING]
    uint64_t* qfull = tkempty + RING;             // [STAGES] int stages land here (by int-stage sequence number)
    uint64_t* qdone = qfull + STAGES;             // [STAGES] every transform warp has read that int stage
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qdone + STAGES);
    int32_t* ent_s = reinterpret_cast<int32_t*>(tmem_slot + 4);           // [64] epilogue: entry ids
    float* gate_s = reinterpret_cast<float*>(ent_s + 64);                 // [64] epilogue: gates
    Tick* ring = reinterpret_cast<Tick*>(gate_s + 64);                    // [RING]

    const int K = PHASE == 0 ? a.H : a.I;
    const int nmb = PHASE == 0 ? a.I / 64 : (a.H + 127) / 128;
    const int nk = K / KCH;
    const int G = K / a.g;
    const bool tab_ok = G <= GTAB;
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < NA; ++b) { mbar_init(&aready[b], 4); mbar_init(&aempty[b], 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4);
            mbar_init(&tabfull[b], 1); mbar_init(&tabempty[b], NTW);
        }
        for (int b = 0; b < RING; ++b) { mbar_init(&tkfull[b], 1); mbar_init(&tkempty[b], N_CONSUMERS); }
        for (int s = 0; s < STAGES; ++s) { mbar_init(&qfull[s], 1); mbar_init(&qdone[s], NTW); }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 3; ++i) tma_prefetch(&mp.b[i][0]);
        tma_prefetch(&mp.a16);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n_act = a.n_act[0];
    const int n_items = n_act * nmb;
    // the active experts' rows, slots and tiers, read once into shared memory so the scheduler decodes a ticket
    // without a dependent chain of global loads per item
    for (int i = threadIdx.x; i < n_act && i < EMAX; i += THREADS) {
        const int e = a.act_e[i];
        const int r0 = a.off[e];
        etab[i] = make_int4(r0, a.off[e + 1] - r0, e < a.E_loc ? a.slot[e] : a.shared_slot, e < a.E_loc ? a.tier[e] : 1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t tmem_a = tmem + 2 * ACC_COLS;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        int st = 0, tc = 0, qs = 0;                  // ring position, int items, int stages issued
        uint32_t ph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, nk, w); ++ii) {
            const bool qt = w.bits != 16 && a.dbg != 12;    // dbg 12 (timing only): int stages flow like bf16 ones
            if ((a.dbg == 9 || a.dbg == 12) && lane == 0) {
                trace(PHASE, ii, 1, globaltimer_ns());
                trace(PHASE, ii, 7, (unsigned long long)w.bits | ((unsigned long long)w.m << 8) | ((unsigned long long)w.nst << 16));
            }
            if (w.bits != 16 && tab_ok) {
                const int tb = tc & 1;
                dwait(&tabempty[tb], ((tc >> 1) & 1) ^ 1, 1);
                ++tc;
                if (elect_one()) {
                    const SlotLayout& L = w.ti ? a.hi : a.lo;
                    const uint8_t* sb = a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
                    uint8_t* ts = tabs + tb * TAB_BYTES;
                    uint8_t* tz = ts + 128 * GTAB * 2;
                    if (PHASE == 0) {
                        const uint32_t sbytes = 64 * G * 2, zbytes = 64 * G;
                        mbar_arrive_expect_tx(&tabfull[tb], 2 * (sbytes + zbytes));
                        const int64_t row = (int64_t)w.mb * 64;
                        for (int m = 0; m < 2; ++m) {        // gate rows -> table rows 0-63, up rows -> 64-127
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
            const CUtensorMap* amap = w.bits != 16 ? &mp.cq[w.ti][w.wi] : &mp.a16;
            const CUtensorMap* bmap = &mp.b[w.rbi][w.ksi];
            const int arow = PHASE == 0 ? w.mb * 64 : w.mb * 128;
            const int kunit = w.bits != 16 ? KCH * w.bits / 8 : KCH;       // A inner coordinate per chunk (bytes / elements)
            const uint32_t abytes = w.bits != 16 ? 128u * (uint32_t)(w.ks * KCH * w.bits / 8) : (uint32_t)A_BYTES;
            const uint32_t bytes = abytes + (uint32_t)(w.ks * w.rb * 128);
            for (int s = 0; s < w.nst; ++s) {
                const int kb0 = s * w.ks;
                // an int stage lands on qfull[qs % STAGES]; that barrier is re-armed only after every transform
                // warp has released its previous use (qdone), so no warp can see a stale phase
                if (qt && qs >= STAGES) dwait(&qdone[qs % STAGES], (uint32_t)((qs / STAGES) - 1) & 1, 12);
                dwait(&empty[st], ph ^ 1, 2);
                if (elect_one()) {
                    uint8_t* sA = sS + st * STAGE_BYTES;
                    uint64_t* fb = qt ? &qfull[qs % STAGES] : &full[st];
                    mbar_arrive_expect_tx(fb, bytes);
                    if (PHASE == 0) tma_load_4d(sA, amap, fb, kb0 * kunit, arow, 0, w.slot);
                    else tma_load_3d(sA, amap, fb, kb0 * kunit, arow, w.slot);
                    tma_load_3d(sA + A_BYTES, bmap, fb, 0, w.r0, kb0);
                    if (qt) mbar_arrive(&full[st]);       // keeps full[]'s phase sequence for the MMA warp
                }
                __syncwarp();
                if (qt) ++qs;
                if (++st == STAGES) { st = 0; ph ^= 1; }
            }
            if ((a.dbg == 9 || a.dbg == 12) && lane == 0) trace(PHASE, ii, 2, globaltimer_ns());
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (lane 0 issues; warp-uniform walk)
        int st = 0, cc = 0, ch = 0;
        uint32_t ph = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, nk, w); ++ii, ++cc) {
            const uint32_t idesc = idesc_bf16(128, w.rb);
            const int buf = cc & 1;
            dwait(&tempty[buf], ((cc >> 1) & 1) ^ 1, 3);
            tc_fence_after();
            const uint32_t d = tmem + buf * ACC_COLS;
            const uint32_t bstep = (w.rb * 128) >> 4;              // B sub-tile stride in descriptor units
            for (int s = 0; s < w.nst; ++s) {
                const int kb0 = s * w.ks;
                const int kc = min(w.ks, nk - kb0);
                dwait(&full[st], ph, 4);
                if ((a.dbg == 9 || a.dbg == 12) && s == 0 && lane == 0) trace(PHASE, ii, 3, globaltimer_ns());
                tc_fence_after();
                const uint32_t sA = smem_u32(sS + st * STAGE_BYTES), sB = sA + A_BYTES;
                const uint64_t db = umma_desc_sw128(sB);
                if (w.bits == 16) {
                    const uint64_t da = umma_desc_sw128(sA);
                    if (elect_one()) {
#pragma unroll
                        for (int q = 0; q < KCH / 16; ++q) mma_bf16(d, da + 2 * q, db + 2 * q, idesc, (kb0 | q) != 0);
                        mma_commit(&empty[st]);
                    }
                    __syncwarp();
                } else if (a.dbg == 12) {
                    if (elect_one()) mma_commit(&empty[st]);
                    __syncwarp();
                } else {
                    // every chunk of the stage dequantised, then one issue region for all of its MMAs
                    for (int j = 0; j < kc; ++j) dwait(&aready[(ch + j) % NA], (uint32_t)((ch + j) / NA) & 1, 5);
                    tc_fence_after();
                    if (elect_one()) {
                        for (int j = 0; j < kc; ++j) {
                            const int b = (ch + j) % NA;
                            const uint32_t at = tmem_a + 32 * b;
                            const uint64_t bj = db + j * bstep;
                            if (a.dbg != 4 && a.dbg != 6) {
#pragma unroll
                                for (int q = 0; q < 4; ++q) mma_bf16_ts(d, at + 8 * q, bj + 2 * q, idesc, (kb0 | j | q) != 0);
                            }
                            mma_commit(&aempty[b]);
                        }
                        mma_commit(&empty[st]);
                    }
                    __syncwarp();
                    ch += kc;
                }
                if (++st == STAGES) { st = 0; ph ^= 1; }
            }
            if ((a.dbg == 9 || a.dbg == 12) && lane == 0) trace(PHASE, ii, 4, globaltimer_ns());
            if (elect_one()) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp < W_EPI) {
        // ------------------------------------------------ dequant (thread = weight row = TMEM lane)
        const int grp = (warp - 2) >> 2;              // 0..NG-1: takes the chunks ch = grp (mod NG)
        const int qa = warp & 3;                      // TMEM lane quarter this warp may access
        const int r = 32 * qa + lane;
        const int mat_rows = PHASE == 0 ? a.I : a.H;
        const uint32_t lane_base = tmem_a + ((uint32_t)(32 * qa) << 16);
        const uint32_t stages_u32 = smem_u32(sS);
        const int gsh = 31 - __clz(a.g);
        uint32_t magic = 0x43004300u;
        asm volatile("" : "+r"(magic));
        int nsd = 0, qs = 0, ch = 0, tc = 0;          // ring position, int stages, int chunks (MMA numbering)
        int pend = -1;                                 // TMEM buffer whose tcgen05.st is in flight, aready not yet signalled
        auto flush = [&]() {
            if (pend >= 0) {
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aready[pend]);
                pend = -1;
            }
        };
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, nk, w); ++ii) {
            if (w.bits == 16) { nsd += w.nst; continue; }    // bf16 items need no transform
            if (a.dbg == 12) {
                if (tab_ok) {
                    dwait(&tabfull[tc & 1], (tc >> 1) & 1, 6);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tabempty[tc & 1]);
                    ++tc;
                }
                continue;
            }
            const int mrow = PHASE == 0 ? w.mb * 64 + (r & 63) : w.mb * 128 + r;
            const bool valid = mrow < mat_rows;
            const SlotLayout& L = w.ti ? a.hi : a.lo;
            const int mat = PHASE == 0 ? (r >> 6) : 2;
            const uint8_t* slot_base =
                a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
            const uint16_t* gscales =
                reinterpret_cast<const uint16_t*>(slot_base + L.scales_off + mat * L.scales_stride) + (int64_t)mrow * G;
            const uint8_t* gzeros = slot_base + L.zeros_off + mat * L.zeros_stride + (int64_t)mrow * G;
            const int tb = tc & 1;
            const uint32_t tsc = smem_u32(tabs + tb * TAB_BYTES) + r * G * 2;
            const uint32_t tze = smem_u32(tabs + tb * TAB_BYTES + 128 * GTAB * 2) + r * G;
            if (tab_ok) dwait(&tabfull[tb], (tc >> 1) & 1, 6);
            auto group_sz = [&](int gi) -> uint32_t {       // (bf16 s) | (bf16(128 + z) << 16)
                if (!valid) return 0x43003f80u;             // rows past the matrix: s = 1, z = 0
                return tab_ok ? lds_u16(tsc + 2 * gi) | ((0x4300u + lds_u8(tze + gi)) << 16)
                              : (uint32_t)gscales[gi] | ((0x4300u + gzeros[gi]) << 16);
            };
            const bool four = w.bits == 4;
            for (int s = 0; s < w.nst; ++s, ++nsd, ++qs) {
                const int kb0 = s * w.ks;
                const int kc = min(w.ks, nk - kb0);
                const int sq = qs % STAGES;
                dwait(&qfull[sq], (uint32_t)(qs / STAGES) & 1, 7);   // every warp observes every int stage
                const uint32_t stage = stages_u32 + (nsd % STAGES) * STAGE_BYTES;
                // my chunks in this stage: ch + j with (ch + j) % NG == grp
                for (int j = (grp - ch % NG + NG) % NG; j < kc; j += NG) {
                    const int cj = ch + j, b = cj % NA;
                    uint32_t wv[32];
                    if (a.dbg != 5 && a.dbg != 6) {
                        const int k0 = (kb0 + j) * KCH;
                        const uint32_t v0 = group_sz(k0 >> gsh);
                        const uint32_t v1 = a.g >= 64 ? v0 : group_sz((k0 + 32) >> gsh);
                        const uint32_t zz0 = (v0 >> 16) * 0x10001u, ss0 = (v0 & 0xFFFFu) * 0x10001u;
                        const uint32_t zz1 = (v1 >> 16) * 0x10001u, ss1 = (v1 & 0xFFFFu) * 0x10001u;
                        if (four) {
                            uint32_t c[8];
                            lds128(code_unit(stage, r, 2 * j, w.wi), c[0], c[1], c[2], c[3]);
                            lds128(code_unit(stage, r, 2 * j + 1, w.wi), c[4], c[5], c[6], c[7]);
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const uint32_t zz = u < 4 ? zz0 : zz1, ss = u < 4 ? ss0 : ss1;
                                wv[4 * u + 0] = deq2(and_or(c[u], 0x000F000Fu, magic), zz, ss);
                                wv[4 * u + 1] = deq2(and_or(c[u] >> 4, 0x000F000Fu, magic), zz, ss);
                                wv[4 * u + 2] = deq2(and_or(c[u] >> 8, 0x000F000Fu, magic), zz, ss);
                                wv[4 * u + 3] = deq2(and_or(c[u] >> 12, 0x000F000Fu, magic), zz, ss);
                            }
                        } else {
                            uint32_t c[4];
                            lds128(code_unit(stage, r, j, w.wi), c[0], c[1], c[2], c[3]);
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t zz = u < 2 ? zz0 : zz1, ss = u < 2 ? ss0 : ss1;
#pragma unroll
                                for (int p = 0; p < 8; ++p)
                                    wv[8 * u + p] = deq2(and_or(c[u] >> (2 * p), 0x00030003u, magic), zz, ss);
                            }
                        }
                    }
                    dwait(&aempty[b], ((uint32_t)(cj / NA) & 1) ^ 1, 8);   // TMEM buffer b drained by its MMAs
                    flush();                                                // the previous chunk's store -> aready
                    if (a.dbg != 5 && a.dbg != 6 && a.dbg != 11) {
                        tc_fence_after();
                        tmem_st32(lane_base + 32 * b, wv);
                    } else if (a.dbg == 11) {                   // timing only: the math without the TMEM store
                        uint32_t acc = 0;
#pragma unroll
                        for (int u = 0; u < 32; ++u) acc ^= wv[u];
                        if (acc == 0x9E3779B9u) a.act[0] = __float2bfloat16_rn(0.f);
                    }
                    pend = b;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&qdone[sq]);     // this warp's reads of the stage's codes are done
                ch += kc;
            }
            flush();                                         // nothing outstanding across an item boundary
            if (tab_ok) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&tabempty[tb]);
                ++tc;
            }
        }
    } else if (warp == W_SCHED) {
        // ------------------------------------------------ scheduler: claim a ticket, decode, publish
        int* ctr = a.sched + 2 * PHASE;
        for (int ii = 0;; ++ii) {
            const int sl = ii % RING;
            dwait(&tkempty[sl], ((ii / RING) & 1) ^ 1, 11);
            int item = 0;
            if (lane == 0) {
                item = atomicAdd(ctr, 1);
                if (a.dbg == 9 || a.dbg == 12) trace(PHASE, ii, 0, globaltimer_ns());
                int4 v = make_int4(0, 0, 0, 0);
                if (item < n_items) {
                    const int i = item / nmb;
                    if (i < EMAX) {
                        v = etab[i];
                    } else {
                        const int e = a.act_e[i];
                        const int r0 = a.off[e];
                        v = make_int4(r0, a.off[e + 1] - r0, e < a.E_loc ? a.slot[e] : a.shared_slot, e < a.E_loc ? a.tier[e] : 1);
                    }
                }
                ring[sl].v = v;
                ring[sl].item = item;
                mbar_arrive(&tkfull[sl]);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= n_items) break;
        }
    } else {
        // ------------------------------------------------ epilogue (4 warps, thread = accumulator lane)
        const int q = warp & 3;
        const int et = threadIdx.x - 32 * W_EPI;
        int cc = 0;
        Item w;
        for (int ii = 0; take_item(a, ring, tkfull, tkempty, ii, n_items, nmb, nk, w); ++ii, ++cc) {
            const int buf = cc & 1;
            const int nvalid = w.m;
            if (PHASE == 1) {
                for (int i = et; i < nvalid; i += 128) {
                    const int ent = a.perm[w.r0 + i];
                    ent_s[i] = ent;
                    gate_s[i] = a.gate[ent];
                }
            }
            dwait(&tfull[buf], (cc >> 1) & 1, 9);
            if ((a.dbg == 9 || a.dbg == 12) && et == 0) trace(PHASE, ii, 5, globaltimer_ns());
            tc_fence_after();
            named_bar(1, 128);
            for (int col = 0; col < (a.dbg == 8 ? 0 : nvalid); col += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + buf * ACC_COLS + ((uint32_t)(32 * q) << 16) + col, v);
                tmem_ld_wait();
                if (PHASE == 0) {
                    // gate rows 0-63 (warps q < 2) meet their up rows 64-127 (q >= 2) through smem; the gate
                    // warps take token columns 0-15 of the block, the up warps 16-31.  a = bf16(silu(g) * u)
                    float* xu = xch;
                    float* xg = xch + 16 * 64;
                    const int rr = 32 * (q & 1) + lane;
                    if (q >= 2) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) xu[j * 64 + rr] = __uint_as_float(v[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) xg[j * 64 + rr] = __uint_as_float(v[16 + j]);
                    }
                    named_bar(1, 128);
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
                    named_bar(1, 128);
                } else {
                    const int h = w.mb * 128 + 32 * q + lane;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (col + j < nvalid && h < a.H) {
                            const int ent = ent_s[col + j];
                            a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(gate_s[col + j] * __uint_as_float(v[j]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if ((a.dbg == 9 || a.dbg == 12) && et == 0) trace(PHASE, ii, 6, globaltimer_ns());
            named_bar(1, 128);                      // ent_s / gate_s / xch reused by the next item
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (threadIdx.x == 0) {                        // the last CTA out resets the ticket counter
        int* ctr = a.sched + 2 * PHASE;
        __threadfence();
        if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(ctr, 0);
            atomicExch(ctr + 1, 0);
        }
    }
}

template <int PHASE>
void launch_dec_one(const DecMaps& lm, const DecBMaps& bm, const DecArgs& a, int items, cudaStream_t st) {
    static unsigned long long attr_mask = 0;
    if (dx_first_on_device(attr_mask))
        cudaFuncSetAttribute(k_dec<PHASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    const int grid = items < DX_NUM_SMS ? items : DX_NUM_SMS;
    DecPhaseMaps mp;
    mp.a16 = lm.a16[PHASE];
    for (int t = 0; t < 2; ++t)
        for (int w = 0; w < 3; ++w) mp.cq[t][w] = lm.cq[t][PHASE][w];
    memcpy(mp.b, bm.b[PHASE], sizeof(mp.b));
    dx_launch(k_dec<PHASE>, dim3(grid), dim3(THREADS), SMEM, st, g_dx_pdl, mp, a);
}

}  // namespace

extern "C" int64_t dx_debug_dec_trace(void* host, int64_t bytes) {   // DX_GEMM_DBG=9 timeline (timing study)
    const int64_t n = (int64_t)sizeof(g_dec_trace);
    if (!host && bytes < 0) {                          // clear
        static unsigned long long zero[sizeof(g_dec_trace) / 8];
        return cudaMemcpyToSymbol(g_dec_trace, zero, n) == cudaSuccess ? 0 : -1;
    }
    if (!host) return n;
    if (bytes < n || cudaMemcpyFromSymbol(host, g_dec_trace, n) != cudaSuccess) return -1;
    return n;
}

static uint32_t* g_dec_trap_host = nullptr;
void dec_trap_init() {
    if (g_dec_trap_host) return;
    if (cudaHostAlloc(reinterpret_cast<void**>(&g_dec_trap_host), 64, cudaHostAllocMapped) != cudaSuccess) {
        g_dec_trap_host = nullptr;
        return;
    }
    memset(g_dec_trap_host, 0, 64);
    uint32_t* dptr = nullptr;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), g_dec_trap_host, 0);
    cudaMemcpyToSymbol(g_dec_trap, &dptr, sizeof(dptr));
    if (const char* w = getenv("DX_WATCHDOG_S")) {
        const uint64_t ns = (uint64_t)(atof(w) * 1e9);
        if (ns > 0) cudaMemcpyToSymbol(g_dec_watchdog_ns, &ns, sizeof(ns));
    }
    if (const char* w = getenv("DX_DEC_BACKOFF")) {
        const int h = atoi(w);
        cudaMemcpyToSymbol(g_dec_backoff_ns, &h, sizeof(h));
    }
    if (const char* w = getenv("DX_DEC_WAIT")) {
        const int h = atoi(w);
        cudaMemcpyToSymbol(g_dec_wait_hint, &h, sizeof(h));
    }
}
static const char* const k_dec_trap_names[] = {"?", "tabempty (producer)", "empty (producer)", "tempty (MMA)", "full (MMA)",
                                               "aready (MMA)", "tabfull (dequant)", "qfull (dequant)", "aempty (dequant)",
                                               "tfull (epilogue)", "tkfull (item ring)", "tkempty (scheduler)",
                                               "qdone (producer)"};
int dec_trap_report(char* buf, size_t n) {
    if (!g_dec_trap_host || (g_dec_trap_host[0] >> 16) != 0xDEADu) return 0;
    const uint32_t tag = g_dec_trap_host[0] & 0xFFFFu;
    return snprintf(buf, n, " [k_dec watchdog: wait on %s, parity %u, block %u, thread %u]",
                    tag < 13 ? k_dec_trap_names[tag] : "?", g_dec_trap_host[1], g_dec_trap_host[2], g_dec_trap_host[3]);
}

void launch_dec(int phase, const DecMaps& lm, const DecBMaps& bm, const DecArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 0) launch_dec_one<0>(lm, bm, a, max_items, st);
    else launch_dec_one<1>(lm, bm, a, max_items, st);
}
