// api.cu -- the C ABI (include/dx.h): pool lifecycle, the MoE layer forward, the controller
// schedule and inspection.  Host logic only; all arithmetic of the path runs in the kernels.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <cmath>
#include <algorithm>
#include <chrono>
#include <fcntl.h>
#include <unistd.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "dx_common.cuh"

void launch_manual(const Ctrl& c, int layer, const int2* cmds, int n, int32_t* status, cudaStream_t st);

bool g_dx_pdl = [] {
    const char* s = getenv("DX_PDL");
    return !(s && s[0] == '0');
}();

static thread_local char g_err[1024] = "";
void dx_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    size_t len = strlen(g_err);
    gemm_trap_report(g_err + len, sizeof(g_err) - len);
    len = strlen(g_err);
}
extern "C" const char* dx_last_error(void) { return g_err; }
extern "C" const char* dx_version(void) { return "dynaexq-b200 0.1 (sm_100a)"; }

#define DX_CHECK(cond, code, ...)      \
    do {                               \
        if (!(cond)) {                 \
            dx_set_error(__VA_ARGS__); \
            return code;               \
        }                              \
    } while (0)

struct dx_pool_s {
    dx_config cfg;
    dx_info info;
    int E, E_loc, e_lo, L, k, H, I, g;
    SlotLayout hi, lo;
    i64 layer_bytes, hi_base;
    uint8_t* arena = nullptr;
    uint8_t* weights = nullptr;
    Ctrl ctrl;
    RouteWs ws;                             // routing of the rows this GPU's experts process
    RouteWs ws_src{};                       // EP: routing of this GPU's own tokens over global experts
    RouteWs ws_src_live{};                  // ws_src as used by the last dispatch (caller idx/gate)
    size_t n_ent = 0;                       // workspace rows
    int ep_T = 0;                           // tokens of the last dispatch (for the combine)
    __nv_bfloat16* act = nullptr;
    __nv_bfloat16* Y = nullptr;
    int32_t* err_flag = nullptr;
    int32_t* dev_err = nullptr;             // sticky device-side error (EP routed rows), reported by dx_sync
    int32_t* dn_done = nullptr;         // fused decode FFN: gate/up items done per active expert (self-resetting)
    int64_t prof_fused = 0;             // profiled forwards whose FFN ran as one fused launch
    int32_t* gemm_sched = nullptr;      // [kernel: k_gemm, k_wide][phase][ticket counter, CTAs done] (self-resetting)
    int2* manual_cmds = nullptr;
    int32_t* manual_status = nullptr;
    const uint8_t** hi_img_dev = nullptr;   // [L * E_loc]
    std::vector<const uint8_t*> hi_img_host;
    uint8_t* hi_cache = nullptr;            // library-owned pinned HIGH images when high_bits < 16
    cudaStream_t cs = nullptr, ss = nullptr;
    bool own_ss = false;
    std::vector<i64> t;                     // host mirror of the fold count per layer
    std::vector<i64> publish_at;            // -1 none
    std::vector<u64> pend_tokens;
    std::vector<int> finalized;
    std::vector<cudaEvent_t> ev_side;
    cudaEvent_t ev_plan = nullptr;
    i64 launches = 0;
    u64 wbytes[2][2];                       // [tier][phase] algorithmic weight bytes per expert
    bool profiling = false;
    int prof_every = 1;                 // profile every prof_every-th forward (event timing + byte counters)
    int64_t prof_ctr = 0;
    std::vector<cudaEvent_t> prof_ev;       // 4 per forward: start, after routing, between FFN phases, end
    std::vector<cudaEvent_t> prof_free;
    std::vector<cudaEvent_t> prof_wait_ev;  // pairs around the publish wait (exposed switch time)
    std::vector<cudaEvent_t> prof_xfer_ev;  // pairs around side-stream transitions (switch latency)
    std::vector<cudaEvent_t> prof_copy_ev;  // pairs around the copy-engine promotions of a plan
    std::vector<u64> prof_copy_bytes;       // their bytes
    cudaStream_t ss2 = nullptr;             // second side stream: demotion kernels beside the H2D copies
    cudaEvent_t ev_dem = nullptr;
    i64 prof_fwd = 0;
    int ffn_path = 0;                       // 0: tcgen05 grouped GEMM, 1: mma.sync decode kernel
    bool last_logits_router = false;        // the last forward computed router logits into ws.logits
    int last_T = 0;
    __nv_bfloat16* Xp = nullptr;            // x rows in permuted order (B operand of gate/up)
    std::vector<GemmMaps> gmaps;            // per layer (weights); xb filled per launch
    CUtensorMap xb0[4], xb1[4];             // B operand maps (Xp / act) for tiles of 16, 32, 64, 128 rows
    CUtensorMap xw0, xw1;                   // the same, 256-row tiles (k_wide)
    CUtensorMap xp0, xp1;                   // the same, 192-row tiles (k_gemm prefill)
    CUtensorMap xk0[3], xk1[3];             // 3-D B maps (Xp / act): several K chunks per box (decode int)
    // expert parallelism over NCCL (ep_nccl.cu): library-owned communicator and exchange buffers
    void* comm = nullptr;
    __nv_bfloat16 *ep_send_rows = nullptr, *ep_recv_rows = nullptr, *ep_y_rows = nullptr, *ep_back_rows = nullptr;
    int4 *ep_send_meta = nullptr, *ep_recv_meta = nullptr;   // per entry {local expert, gate bits, row in block}
    int2* ep_meta2 = nullptr;               // owner side: {expert, gate} of the received entries
    int32_t* ep_rowmap = nullptr;           // owner side: the received row of each received entry (f-2)
    int32_t* ep_mark = nullptr;             // source side: [G][T] dedup marks -> rows within owner blocks
    int32_t* ep_pairs = nullptr;            // device [2][G][3]: my {unique rows, entries, T} per peer | received
    int32_t* ep_pairs_host = nullptr;       // pinned mirror (the v1 host synchronisation point)
    bool ep_group = false;                  // EP buffers without a communicator: member of a local pool group
    u64 ep_rows_sent = 0, ep_entries_sent = 0;   // f-2 accounting (rows actually moved vs one row per entry)
    u64 copy_promotions = 0;                // promotions issued as copy-engine H2D copies
    // f-4 SSD tier (dx_pool_create_ssd): every HIGH image in one file, a pinned DRAM cache of `ssd_slots` images
    // in front of it (LRU; a slot is reused only after the copies out of it completed)
    int ssd_fd = -1;
    std::string ssd_path;
    bool ssd_direct = false;
    int ssd_slots = 0;
    size_t img_bytes = 0;                   // bytes of one HIGH image (the promotion copy size)
    uint8_t* ssd_cache = nullptr;           // pinned [ssd_slots][img_bytes]
    std::vector<int> cache_slot_of;         // [L * E_loc] -> slot or -1
    std::vector<int> cache_owner;           // [slot] -> key or -1
    std::vector<u64> cache_used;            // [slot] LRU clock
    std::vector<cudaEvent_t> cache_ev;      // [slot] last copy out of the slot
    u64 cache_clock = 0, ssd_reads = 0, ssd_bytes = 0, cache_hits = 0;
    double ssd_read_ms = 0.0;
    // SSD reads of runtime plans run on an I/O thread so the issuing host thread never blocks on the device: it
    // hands over {layer, copies}; the worker reads, copies on the side stream and records the layer's ev_side;
    // publication waits for the hand-over to finish before waiting on ev_side.  The cache is guarded by io_mu.
    struct IoJob {
        int layer;
        std::vector<std::pair<size_t, uint8_t*>> copies;
        bool wait_dem;
        cudaEvent_t xc, x1;
    };
    int device = 0;
    std::thread io_thread;
    std::mutex io_mu;
    std::condition_variable io_cv;
    std::deque<IoJob> io_q;
    std::vector<int> io_pending;            // per layer: a job handed over and not finished
    int io_inflight = 0;
    bool io_stop = false;
    dx_status io_err = DX_OK;
    // f-1 cross-layer correlation prefetch (dx_set_prefetch): device counts per layer pair, the last routing of
    // each layer parity, candidates staged into free HIGH blocks ahead of the plan
    uint32_t* corr = nullptr;               // [L-1][E][E]
    int32_t* idx_last = nullptr;            // [2][max_tokens * k]
    int T_last[2] = {-1, -1};
    int pf_f = 0, pf_lead = 0;
    int4* pf_dev = nullptr;                 // [L][8]
    int32_t* pf_n_dev = nullptr;            // [L]
    int4* pf_host = nullptr;                // pinned mirror
    int32_t* pf_n_host = nullptr;
    std::vector<cudaEvent_t> ev_pf;
    std::vector<int> pf_pending;
    std::vector<std::vector<int2>> staged;  // per layer: {expert, block} copies issued for the coming plan
    u64 pf_issued = 0, pf_hits = 0;
    bool teleport = false;                  // timing baseline: plans and publications without the transfers
    int hi_slots = 1;                       // HIGH blocks addressable by the tensor maps (incl. the shared one)
    int shared_slot = 0;                    // f-3: the shared expert's HIGH block index
    // runtime plans reach the host through pinned memory; the host then issues the promotions' H2D copies on the
    // copy engine (cudaMemcpyAsync on the side stream) and the demotion kernel -- as soon as the plan is seen
    // done (polled at every library call), at the latest at the publication step
    int4* plan_host = nullptr;              // pinned [L][E_loc] copy of the device plan list
    int32_t* plan_n_host = nullptr;         // pinned [L]
    std::vector<cudaEvent_t> ev_planh;      // plan copied to the host
    std::vector<cudaEvent_t> ev_plandone;   // plan kernel done (compute stream): the side stream copies the plan out
    std::vector<int> xfer_pending;          // per layer: plan made, transfers not yet issued
    int n_pending = 0;
                                            // configuration (A/B runs; measured slower on the int tiers)
};

// ---------------------------------------------------------------- TMA tensor maps (driver entry point)
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static bool get_encode() {
    if (g_encode) return true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        cudaGetLastError();
        return false;
    }
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return true;
}
static bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                     const uint64_t* strides, const uint32_t* box, CUtensorMapSwizzle sw) {
    uint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(m, dt, rank, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static dx_status build_maps(dx_pool p) {
    if (!get_encode()) { dx_set_error("cuTensorMapEncodeTiled unavailable"); return DX_ERR_CUDA; }
    const int H = p->H, I = p->I, E = p->E_loc, s = p->cfg.n_spare, T = p->cfg.max_tokens, k = p->k;
    const int cap_hi = p->info.cap_hi;
    p->gmaps.assign(p->L, GemmMaps{});
    for (int l = 0; l < p->L; ++l) {
        GemmMaps& g = p->gmaps[l];
        const uint8_t* lb = p->weights + (size_t)l * p->layer_bytes;
        bool ok = true;
        if (p->hi.bits == 16) {
            const uint64_t d0[4] = {(uint64_t)H, (uint64_t)I, 2, (uint64_t)p->hi_slots};
            const uint64_t s0[3] = {(uint64_t)H * 2, (uint64_t)p->hi.codes_stride, (uint64_t)p->hi.bytes};
            const uint32_t b0[4] = {64, 64, 2, 1};           // 64 gate rows, then the 64 matching up rows
            ok &= make_map(&g.a16_gu, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, lb + p->hi_base, d0, s0, b0,
                           CU_TENSOR_MAP_SWIZZLE_128B);
            const uint64_t d1[3] = {(uint64_t)I, (uint64_t)H, (uint64_t)p->hi_slots};
            const uint64_t s1[2] = {(uint64_t)I * 2, (uint64_t)p->hi.bytes};
            const uint32_t b1[3] = {64, 128, 1};
            ok &= make_map(&g.a16_dn, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, lb + p->hi_base + (size_t)2 * I * H * 2, d1, s1,
                           b1, CU_TENSOR_MAP_SWIZZLE_128B);
        }
        for (int t = 0; t < 2; ++t) {
            const SlotLayout& Ls = t ? p->hi : p->lo;
            if (Ls.bits == 16) continue;
            const uint8_t* base = lb + (t ? p->hi_base : 0);
            const uint64_t slots = t ? (uint64_t)p->hi_slots : (uint64_t)(E + s);
            const uint64_t rb0 = (uint64_t)H * Ls.bits / 8, rb1 = (uint64_t)I * Ls.bits / 8;
            const uint32_t kb = 64 * Ls.bits / 8;
            const uint64_t d0[4] = {rb0, (uint64_t)I, 2, slots};
            const uint64_t s0[3] = {rb0, (uint64_t)Ls.codes_stride, (uint64_t)Ls.bytes};
            const uint32_t b0[4] = {kb, 64, 2, 1};
            ok &= make_map(t ? &g.ahi_gu : &g.alo_gu, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, d0, s0, b0,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
            const uint64_t d1[3] = {rb1, (uint64_t)H, slots};
            const uint64_t s1[2] = {rb1, (uint64_t)Ls.bytes};
            const uint32_t b1[3] = {kb, 128, 1};
            ok &= make_map(t ? &g.ahi_dn : &g.alo_dn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base + 2 * Ls.codes_stride, d1, s1,
                           b1, CU_TENSOR_MAP_SWIZZLE_NONE);
            // decode stages: 128 B of codes per row (16 / bits K chunks) in one box; the tail past the row
            // end is zero-filled by TMA and never read
            const uint32_t w0[4] = {128, 64, 2, 1}, w1[3] = {128, 128, 1};
            ok &= make_map(t ? &g.whi_gu : &g.wlo_gu, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, d0, s0, w0,
                           CU_TENSOR_MAP_SWIZZLE_128B);
            ok &= make_map(t ? &g.whi_dn : &g.wlo_dn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base + 2 * Ls.codes_stride, d1, s1,
                           w1, CU_TENSOR_MAP_SWIZZLE_128B);
        }
        if (!ok) { dx_set_error("tensor map encoding failed (layer %d)", l); return DX_ERR_CUDA; }
    }
    for (int i = 0; i < 4; ++i) {
        const uint32_t bn = 16u << i;                       // B tile rows 16, 32, 64, 128
        const uint64_t rows = (uint64_t)p->n_ent;
        (void)T; (void)k;
        const uint64_t d0[2] = {(uint64_t)H, rows}, s0[1] = {(uint64_t)H * 2};
        const uint64_t d1[2] = {(uint64_t)I, rows}, s1[1] = {(uint64_t)I * 2};
        const uint32_t b[2] = {64, bn};
        const uint32_t bw[2] = {64, 256}, bp[2] = {64, 192};
        if (!make_map(&p->xb0[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->Xp, d0, s0, b, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_map(&p->xb1[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->act, d1, s1, b, CU_TENSOR_MAP_SWIZZLE_128B) ||
            (i == 0 && (!make_map(&p->xw0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->Xp, d0, s0, bw, CU_TENSOR_MAP_SWIZZLE_128B) ||
                        !make_map(&p->xw1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->act, d1, s1, bw, CU_TENSOR_MAP_SWIZZLE_128B) ||
                        !make_map(&p->xp0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->Xp, d0, s0, bp, CU_TENSOR_MAP_SWIZZLE_128B) ||
                        !make_map(&p->xp1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->act, d1, s1, bp, CU_TENSOR_MAP_SWIZZLE_128B)))) {
            dx_set_error("tensor map encoding failed (activations)");
            return DX_ERR_CUDA;
        }
    }
    for (int i = 0; i < 3; ++i) {                           // {rows, chunks}: {16, 4}, {32, 4}, {16, 8}
        const uint32_t bn = i == 1 ? 32 : 16, nc = i == 2 ? 8 : 4;
        const uint64_t rows = (uint64_t)p->n_ent;
        const uint64_t d0[3] = {64, rows, (uint64_t)H / 64}, s0[2] = {(uint64_t)H * 2, 128};
        const uint64_t d1[3] = {64, rows, (uint64_t)I / 64}, s1[2] = {(uint64_t)I * 2, 128};
        const uint32_t b[3] = {64, bn, nc};
        if (!make_map(&p->xk0[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->Xp, d0, s0, b, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_map(&p->xk1[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->act, d1, s1, b, CU_TENSOR_MAP_SWIZZLE_128B)) {
            dx_set_error("tensor map encoding failed (activations, 3-D)");
            return DX_ERR_CUDA;
        }
    }
    return DX_OK;
}

static cudaEvent_t prof_event(dx_pool p) {
    if (p->prof_free.empty()) {
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = p->prof_free.back();
    p->prof_free.pop_back();
    return e;
}

static u64 phase_bytes(const SlotLayout& L, int H, int I, int g, int nmat) {
    const u64 n = (u64)I * H;
    if (L.bits == 16) return nmat * n * 2;
    return nmat * (n * L.bits / 8 + n / g * 3);
}

static int64_t slot_bytes_impl(int H, int I, int g, int bits) { return dx_slot_layout(H, I, g, bits).bytes; }

extern "C" int64_t dx_slot_bytes(int32_t H, int32_t I, int32_t g, int32_t bits) {
    if (H <= 0 || I <= 0 || g <= 0 || (bits != 16 && bits != 4 && bits != 2)) return -1;
    return slot_bytes_impl(H, I, g, bits);
}

extern "C" int64_t dx_solve_n_hot(int64_t M, int32_t N, int64_t S_h, int64_t S_l, int32_t s) {
    // largest n_hot with (n_hot+s) S_h + (N-n_hot+s) S_l <= M  (R-P2)
    const int64_t num = M - (int64_t)N * S_l - (int64_t)s * (S_h + S_l);
    if (num < 0 || S_h <= S_l) return -1;
    const int64_t n = num / (S_h - S_l);
    return n < N ? n : N;
}

template <typename T>
static T* carve(uint8_t*& p, size_t count) {
    uintptr_t a = ((uintptr_t)p + 255) & ~(uintptr_t)255;
    T* r = reinterpret_cast<T*>(a);
    p = reinterpret_cast<uint8_t*>(a + count * sizeof(T));
    return r;
}

static dx_status validate(const dx_config* c) {
    DX_CHECK(c, DX_ERR_INVALID_ARG, "null config");
    DX_CHECK(c->num_layers >= 1 && c->num_experts >= 1, DX_ERR_INVALID_ARG, "num_layers/num_experts must be >= 1");
    DX_CHECK(c->top_k >= 1 && c->top_k <= c->num_experts && c->top_k <= 16, DX_ERR_INVALID_ARG,
             "top_k must be in [1, min(E, 16)]");
    DX_CHECK(c->group_size == 32 || c->group_size == 64 || c->group_size == 128, DX_ERR_INVALID_ARG,
             "group_size must be 32, 64 or 128");
    DX_CHECK(c->hidden % 64 == 0 && c->inter % 64 == 0 && c->hidden % c->group_size == 0 &&
             c->inter % c->group_size == 0 && c->hidden > 0 && c->inter > 0,
             DX_ERR_INVALID_ARG, "hidden/inter must be positive multiples of 64 and of group_size");
    DX_CHECK((c->high_bits == 16 && (c->low_bits == 4 || c->low_bits == 2)) || (c->high_bits == 4 && c->low_bits == 2),
             DX_ERR_INVALID_ARG, "precision pair must be (16,4), (16,2) or (4,2)");
    DX_CHECK(c->ema_alpha > 0.0 && c->ema_alpha < 1.0, DX_ERR_INVALID_ARG, "ema_alpha in (0,1)");
    DX_CHECK(c->period >= 1 && c->warmup_steps >= 0 && c->dwell_min >= 0 && c->n_spare >= 0, DX_ERR_INVALID_ARG,
             "period >= 1, warmup >= 0, dwell >= 0, n_spare >= 0");
    DX_CHECK(c->publish_lag >= 1 && c->publish_lag < c->period, DX_ERR_INVALID_ARG, "1 <= publish_lag < period");
    DX_CHECK(c->max_tokens >= 1, DX_ERR_INVALID_ARG, "max_tokens >= 1");
    DX_CHECK(c->ep_size >= 1 && c->ep_rank >= 0 && c->ep_rank < c->ep_size && c->num_experts % c->ep_size == 0,
             DX_ERR_INVALID_ARG, "ep_size must divide num_experts and 0 <= ep_rank < ep_size");
    DX_CHECK(c->num_experts <= 512 && c->num_experts + c->n_spare <= 1024, DX_ERR_INVALID_ARG,
             "num_experts must be <= 512");
    DX_CHECK(c->n_shared == 0 || c->n_shared == 1, DX_ERR_INVALID_ARG, "n_shared must be 0 or 1");
    DX_CHECK(c->n_shared == 0 || c->ep_size == 1, DX_ERR_INVALID_ARG, "a shared expert needs ep_size == 1");
    return DX_OK;
}

// ---------------------------------------------------------------- f-4 SSD tier
static dx_status ssd_write(dx_pool p, size_t key, const void* src) {
    const uint8_t* b = static_cast<const uint8_t*>(src);
    size_t done = 0;
    while (done < p->img_bytes) {
        const ssize_t r = pwrite(p->ssd_fd, b + done, p->img_bytes - done, (off_t)(key * p->img_bytes + done));
        DX_CHECK(r > 0, DX_ERR_INVALID_ARG, "SSD tier write failed (expert image %zu)", key);
        done += (size_t)r;
    }
    return DX_OK;
}

// The pinned host image of HIGH image `key` = layer * E_loc + expert: a DRAM-cache hit, or an SSD read into the
// least recently used slot (after the copies out of that slot completed).  *slot_out: the cache slot.
static dx_status cached_image(dx_pool p, size_t key, const uint8_t** img, int* slot_out) {
    int sl = p->cache_slot_of[key];
    if (sl >= 0) {
        ++p->cache_hits;
    } else {
        sl = -1;
        for (int i = 0; i < p->ssd_slots && sl < 0; ++i)
            if (p->cache_owner[i] < 0) sl = i;                      // a free slot first
        if (sl < 0) {                                              // else the least recently used
            sl = 0;
            for (int i = 1; i < p->ssd_slots; ++i)
                if (p->cache_used[i] < p->cache_used[sl]) sl = i;
        }
        DX_CUDA(cudaEventSynchronize(p->cache_ev[sl]));            // copies out of the victim slot are done
        if (p->cache_owner[sl] >= 0) p->cache_slot_of[(size_t)p->cache_owner[sl]] = -1;
        uint8_t* dst = p->ssd_cache + (size_t)sl * p->img_bytes;
        const auto t0 = std::chrono::steady_clock::now();
        size_t done = 0;
        while (done < p->img_bytes) {
            const ssize_t r = pread(p->ssd_fd, dst + done, p->img_bytes - done, (off_t)(key * p->img_bytes + done));
            DX_CHECK(r > 0, DX_ERR_INVALID_ARG, "SSD tier read failed (expert image %zu)", key);
            done += (size_t)r;
        }
        p->ssd_read_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++p->ssd_reads;
        p->ssd_bytes += p->img_bytes;
        p->cache_owner[sl] = (int)key;
        p->cache_slot_of[key] = sl;
    }
    p->cache_used[sl] = ++p->cache_clock;
    *img = p->ssd_cache + (size_t)sl * p->img_bytes;
    *slot_out = sl;
    return DX_OK;
}

// H2D of HIGH image `key` into a HIGH block on `st` (copy engine): from the pinned masters / HIGH cache, or through
// the SSD tier's DRAM cache
static dx_status copy_high_image(dx_pool p, size_t key, uint8_t* dst, cudaStream_t st) {
    if (p->ssd_fd < 0) {
        DX_CUDA(cudaMemcpyAsync(dst, p->hi_img_host[key], p->img_bytes, cudaMemcpyHostToDevice, st));
        return DX_OK;
    }
    const uint8_t* img;
    int sl;
    std::lock_guard<std::mutex> lk(p->io_mu);
    dx_status rc = cached_image(p, key, &img, &sl);
    if (rc != DX_OK) return rc;
    DX_CUDA(cudaMemcpyAsync(dst, img, p->img_bytes, cudaMemcpyHostToDevice, st));
    DX_CUDA(cudaEventRecord(p->cache_ev[sl], st));
    return DX_OK;
}

static void io_worker(dx_pool p) {
    cudaSetDevice(p->device);
    for (;;) {
        dx_pool_s::IoJob job;
        {
            std::unique_lock<std::mutex> lk(p->io_mu);
            p->io_cv.wait(lk, [&] { return p->io_stop || !p->io_q.empty(); });
            if (p->io_q.empty()) return;
            job = std::move(p->io_q.front());
            p->io_q.pop_front();
        }
        dx_status st = DX_OK;
        for (auto& c : job.copies) {
            if (p->ssd_fd < 0) {             // DRAM tier: the pinned HIGH image straight to its block
                if (cudaMemcpyAsync(c.second, p->hi_img_host[c.first], p->img_bytes, cudaMemcpyHostToDevice, p->ss) !=
                    cudaSuccess) { st = DX_ERR_CUDA; break; }
                continue;
            }
            std::lock_guard<std::mutex> lk(p->io_mu);
            const uint8_t* img;
            int sl;
            st = cached_image(p, c.first, &img, &sl);
            if (st != DX_OK) break;
            if (cudaMemcpyAsync(c.second, img, p->img_bytes, cudaMemcpyHostToDevice, p->ss) != cudaSuccess ||
                cudaEventRecord(p->cache_ev[sl], p->ss) != cudaSuccess) { st = DX_ERR_CUDA; break; }
        }
        if (job.xc) cudaEventRecord(job.xc, p->ss);
        if (job.wait_dem) cudaStreamWaitEvent(p->ss, p->ev_dem, 0);
        if (job.x1) cudaEventRecord(job.x1, p->ss);
        cudaEventRecord(p->ev_side[job.layer], p->ss);
        {
            std::lock_guard<std::mutex> lk(p->io_mu);
            if (st != DX_OK && p->io_err == DX_OK) p->io_err = st;
            p->io_pending[job.layer] = 0;
            --p->io_inflight;
        }
        p->io_cv.notify_all();
    }
}

// the I/O worker finished the layer's hand-over (or, layer < 0, every hand-over); its first error, if any
static dx_status io_wait(dx_pool p, int layer) {
    if (!p->io_thread.joinable()) return DX_OK;
    std::unique_lock<std::mutex> lk(p->io_mu);
    p->io_cv.wait(lk, [&] { return layer >= 0 ? p->io_pending[layer] == 0 : p->io_inflight == 0; });
    const dx_status e = p->io_err;
    p->io_err = DX_OK;
    if (e != DX_OK) dx_set_error("SSD tier: a background read or copy failed");
    return e;
}

static dx_status pool_create(const dx_config* cfg, const void* const* master, void* compute_stream,
                             void* side_stream, const void* nccl_id, dx_pool* out, const char* ssd_path = nullptr,
                             int ssd_slots = 0, bool ep_group = false) {
    dx_status st = validate(cfg);
    if (st != DX_OK) return st;
    DX_CHECK(master && out, DX_ERR_INVALID_ARG, "null master/out");
    dx_pool p = new dx_pool_s();
    p->cfg = *cfg;
    p->L = cfg->num_layers;
    p->E = cfg->num_experts;
    p->E_loc = cfg->num_experts / cfg->ep_size;
    p->e_lo = cfg->ep_rank * p->E_loc;
    p->k = cfg->top_k;
    p->H = cfg->hidden;
    p->I = cfg->inter;
    p->g = cfg->group_size;
    p->hi = dx_slot_layout(p->H, p->I, p->g, cfg->high_bits);
    p->lo = dx_slot_layout(p->H, p->I, p->g, cfg->low_bits);
    const int E = p->E_loc, s = cfg->n_spare;
    const i64 M = (i64)(cfg->expert_budget_bytes / (uint64_t)cfg->num_layers);
    const i64 n_hot = dx_solve_n_hot(M, E, p->hi.bytes, p->lo.bytes, s);
    if (n_hot < 0) {
        dx_set_error("infeasible budget: per-layer %lld B < (N+s)*S_l + s*S_h = %lld B", (long long)M,
                     (long long)((E + s) * p->lo.bytes + s * p->hi.bytes));
        delete p;
        return DX_ERR_INFEASIBLE_BUDGET;
    }
    const int cap_lo = E - (int)n_hot + s, cap_hi = (int)n_hot + s;
    p->hi_base = (i64)cap_lo * p->lo.bytes;
    i64 lb = p->hi_base + (i64)cap_hi * p->hi.bytes;
    if ((i64)E * p->lo.bytes > lb) lb = (i64)E * p->lo.bytes;   // warm-up layout (R-P3)
    p->hi_slots = cap_hi > 0 ? cap_hi : 1;
    if (cfg->n_shared) {
        // f-3: the shared expert's HIGH block after everything else (never part of the warm-up LOW region)
        p->shared_slot = (int)((lb - p->hi_base + p->hi.bytes - 1) / p->hi.bytes);
        p->hi_slots = p->shared_slot + 1;
        lb = p->hi_base + (i64)p->hi_slots * p->hi.bytes;
    }
    p->layer_bytes = dx_up(lb, 1024);

    // ---- the one device allocation: weights | controller | workspace | staging
    const int T = cfg->max_tokens, k = p->k, L = p->L;
    const int G = cfg->ep_size;
    const bool ep_bufs = nccl_id != nullptr || ep_group;   // exchange buffers (NCCL or a local pool group)
    const bool ep = G > 1 || ep_bufs;                // dispatch-side workspace
    // entries (rows) one forward can see: T*k locally; an EP owner receives up to G*T*min(k, E_loc) rows
    const int ns = cfg->n_shared;              // f-3: the shared expert's T rows follow the T*k routed entries
    const size_t n_ent = G > 1 ? std::max((size_t)T * k, (size_t)G * T * std::min(k, E)) : (size_t)T * (k + ns);
    p->n_ent = n_ent;
    const int nblk = route_blocks((int)(ep ? n_ent : (size_t)T));   // the owner side routes up to n_ent rows
    const size_t Ek = (size_t)E;
    size_t ctrl_bytes = 0;
    {
        const size_t LE = (size_t)L * Ek, LO = (size_t)L * (Ek + s);
        ctrl_bytes = LE * (4 + 4 + 4 + 8 + 4 + 8 + 8 + 4 + 4 + 8 + 16) + LO * 8 + L * (8 + 8 + 4 * 3) + 64 * 256;
    }
    const size_t lg_rows = (size_t)T;
    size_t ws_bytes = lg_rows * p->E * 4 + n_ent * (4 + 4 + 4 + 4 + 2 + 4) + 3 * 256 + (size_t)nblk * p->E * 8 +
                      (size_t)(p->E + 1) * 8 + n_ent * (p->I + 2 * p->H) * 2 + 64 * 256 + 4096 * 8 + 256;
    if (ep)      // dispatch-side routing workspace (global experts, local tokens)
        ws_bytes += lg_rows * p->E * 4 + (size_t)T * k * 22 + 3 * 256 + (size_t)route_blocks(T) * p->E * 8 +
                    (size_t)(p->E + 1) * 8 + (size_t)p->E * 4 + 64 * 256;
    if (ep_bufs) // EP exchange buffers: send / back rows (T*k), receive / result rows (n_ent), metadata, counts, marks
        ws_bytes += (size_t)T * k * (2 * p->H * 2 + 16) + n_ent * (2 * p->H * 2 + 16 + 8 + 4) + (size_t)G * 24 +
                    (size_t)G * T * 4 + 8 * 256;
    const size_t stage_bytes = (size_t)3 * p->I * p->H * 2 + p->hi.bytes + 2048 +
                               (size_t)(L > 1 ? L - 1 : 0) * E * E * 4 + (size_t)2 * T * k * 4 + (size_t)L * (8 * 16 + 4) + 4 * 256;
    const size_t ptr_bytes = (size_t)L * E * sizeof(void*) + 256;
    const size_t total = (size_t)L * p->layer_bytes + ctrl_bytes + ws_bytes + stage_bytes + ptr_bytes + 4096;
    cudaError_t ce = cudaMalloc(&p->arena, total);
    if (ce != cudaSuccess) {
        dx_set_error("cudaMalloc(%zu) failed: %s", total, cudaGetErrorString(ce));
        delete p;
        return DX_ERR_OOM;
    }
    uint8_t* q = p->arena;
    p->weights = q;
    q += (size_t)L * p->layer_bytes;
    Ctrl& c = p->ctrl;
    const size_t LE = (size_t)L * E, LO = (size_t)L * (E + s);
    c.tier = carve<int32_t>(q, LE);
    c.slot = carve<int32_t>(q, LE);
    c.version = carve<uint32_t>(q, LE);
    c.S = carve<double>(q, LE);
    c.cnt = carve<uint32_t>(q, LE);
    c.mass = carve<u64>(q, LE);
    c.last = carve<i64>(q, LE);
    c.pend_dir = carve<int32_t>(q, LE);
    c.pend_dst = carve<int32_t>(q, LE);
    c.pend_at = carve<i64>(q, LE);
    c.plan_cmd = carve<int4>(q, LE);
    c.lo_owner = carve<int32_t>(q, LO);
    c.hi_owner = carve<int32_t>(q, LO);
    c.t = carve<i64>(q, L);
    c.tau = carve<double>(q, L);
    c.cap_lo = carve<int32_t>(q, L);
    c.cap_hi = carve<int32_t>(q, L);
    c.plan_n = carve<int32_t>(q, L);
    c.tstats = carve<u64>(q, 2);
    c.E = E; c.s = s; c.n_hot = (int)n_hot; c.W = cfg->warmup_steps; c.Tp = cfg->period;
    c.dwell = cfg->dwell_min; c.lag = cfg->publish_lag; c.alpha = cfg->ema_alpha;
    RouteWs& w = p->ws;
    w.logits = carve<float>(q, lg_rows * p->E);
    w.idx = carve<int32_t>(q, n_ent);
    w.gate = carve<float>(q, n_ent);
    w.hist = carve<int32_t>(q, (size_t)nblk * p->E);
    w.base = carve<int32_t>(q, (size_t)nblk * p->E);
    w.off = carve<int32_t>(q, p->E + 1 + ns);
    w.act_e = carve<int32_t>(q, p->E + ns);
    w.n_act = carve<int32_t>(q, 1);
    w.perm = carve<int32_t>(q, n_ent);
    w.inv = carve<int32_t>(q, n_ent);
    w.stats = carve<u64>(q, 4);
    w.done = carve<unsigned>(q, 1);
    w.ent = carve<int16_t>(q, n_ent);
    w.gm = carve<uint32_t>(q, n_ent);
    w.gbar = carve<unsigned>(q, 2);
    if (ep) {
        RouteWs& v = p->ws_src;
        v.logits = carve<float>(q, lg_rows * p->E);
        v.idx = carve<int32_t>(q, (size_t)T * k);
        v.gate = carve<float>(q, (size_t)T * k);
        v.hist = carve<int32_t>(q, (size_t)route_blocks(T) * p->E);
        v.base = carve<int32_t>(q, (size_t)route_blocks(T) * p->E);
        v.off = carve<int32_t>(q, p->E + 1);
        v.act_e = carve<int32_t>(q, p->E);
        v.n_act = carve<int32_t>(q, 1);
        v.perm = carve<int32_t>(q, (size_t)T * k);
        v.inv = carve<int32_t>(q, (size_t)T * k);
        v.stats = nullptr;
        v.done = carve<unsigned>(q, 1);
        v.ent = carve<int16_t>(q, (size_t)T * k);
        v.gm = carve<uint32_t>(q, (size_t)T * k);
        v.gbar = carve<unsigned>(q, 2);
    }
    if (ep_bufs) {
        p->ep_send_rows = carve<__nv_bfloat16>(q, (size_t)T * k * p->H);
        p->ep_back_rows = carve<__nv_bfloat16>(q, (size_t)T * k * p->H);
        p->ep_send_meta = carve<int4>(q, (size_t)T * k);
        p->ep_recv_rows = carve<__nv_bfloat16>(q, n_ent * p->H);
        p->ep_y_rows = carve<__nv_bfloat16>(q, n_ent * p->H);
        p->ep_recv_meta = carve<int4>(q, n_ent);
        p->ep_meta2 = carve<int2>(q, n_ent);
        p->ep_rowmap = carve<int32_t>(q, n_ent);
        p->ep_mark = carve<int32_t>(q, (size_t)G * T);
        p->ep_pairs = carve<int32_t>(q, (size_t)6 * G);
        p->ep_group = ep_group;
    }
    p->act = carve<__nv_bfloat16>(q, n_ent * p->I);
    p->Y = carve<__nv_bfloat16>(q, n_ent * p->H);
    p->Xp = carve<__nv_bfloat16>(q, n_ent * p->H);
    p->err_flag = carve<int32_t>(q, 1);
    p->dev_err = carve<int32_t>(q, 1);
    p->gemm_sched = carve<int32_t>(q, 12);
    p->dn_done = carve<int32_t>(q, (size_t)p->E_loc + 64);
    p->manual_cmds = carve<int2>(q, 1024);
    p->manual_status = carve<int32_t>(q, 1024);
    p->corr = carve<uint32_t>(q, (size_t)(L > 1 ? L - 1 : 0) * E * E);
    p->idx_last = carve<int32_t>(q, (size_t)2 * T * k);
    p->pf_dev = carve<int4>(q, (size_t)L * 8);
    p->pf_n_dev = carve<int32_t>(q, (size_t)L);
    uint8_t* stage_master = carve<uint8_t>(q, (size_t)3 * p->I * p->H * 2);
    uint8_t* stage_high = carve<uint8_t>(q, (size_t)p->hi.bytes);
    p->hi_img_dev = carve<const uint8_t*>(q, (size_t)L * E);
    if ((size_t)(q - p->arena) > total) {
        dx_set_error("internal: arena carve overflow");
        cudaFree(p->arena);
        delete p;
        return DX_ERR_OOM;
    }

    // ---- streams / events
    p->cs = (cudaStream_t)compute_stream;
    if (side_stream) {
        p->ss = (cudaStream_t)side_stream;
    } else {
        int lo_prio, hi_prio;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        cudaStreamCreateWithPriority(&p->ss, cudaStreamNonBlocking, lo_prio);
        p->own_ss = true;
    }
    cudaEventCreateWithFlags(&p->ev_plan, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p->ev_dem, cudaEventDisableTiming);
    {
        int lo_prio, hi_prio;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        cudaStreamCreateWithPriority(&p->ss2, cudaStreamNonBlocking, lo_prio);
    }
    p->ev_side.resize(L);
    for (int l = 0; l < L; ++l) cudaEventCreateWithFlags(&p->ev_side[l], cudaEventDisableTiming);
    p->ev_planh.resize(L);
    for (int l = 0; l < L; ++l) cudaEventCreateWithFlags(&p->ev_planh[l], cudaEventDisableTiming);
    p->ev_plandone.resize(L);
    for (int l = 0; l < L; ++l) cudaEventCreateWithFlags(&p->ev_plandone[l], cudaEventDisableTiming);
    p->xfer_pending.assign(L, 0);
    p->t.assign(L, 0);
    p->publish_at.assign(L, -1);
    p->pend_tokens.assign(L, 0);
    p->finalized.assign(L, 0);

    auto fail = [&](dx_status code) {
        dx_pool_destroy(p);
        return code;
    };
    p->ev_pf.resize(L);
    for (int l = 0; l < L; ++l) cudaEventCreateWithFlags(&p->ev_pf[l], cudaEventDisableTiming);
    p->pf_pending.assign(L, 0);
    p->staged.assign(L, {});
    if (cudaHostAlloc((void**)&p->pf_host, (size_t)L * 8 * sizeof(int4), cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc((void**)&p->pf_n_host, (size_t)L * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess) {
        dx_set_error("cudaHostAlloc(prefetch mirror) failed");
        return fail(DX_ERR_OOM);
    }
    if (cudaHostAlloc((void**)&p->plan_host, (size_t)L * E * sizeof(int4), cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc((void**)&p->plan_n_host, (size_t)L * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess) {
        dx_set_error("cudaHostAlloc(plan mirror) failed");
        return fail(DX_ERR_OOM);
    }
    if (ep_bufs) {
        if (cudaHostAlloc((void**)&p->ep_pairs_host, (size_t)6 * G * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess) {
            dx_set_error("cudaHostAlloc(EP counts) failed");
            return fail(DX_ERR_OOM);
        }
    }
    if (nccl_id) {
        // collective: every rank of the EP group creates its pool with the same id (blocks until all joined)
        st = ep_nccl_init(nccl_id, G, cfg->ep_rank, &p->comm);
        if (st != DX_OK) return fail(st);
    }

    // ---- HIGH image sources (the DRAM cache)
    p->img_bytes = p->hi.bits == 16 ? (size_t)3 * p->I * p->H * 2 : (size_t)p->hi.bytes;
    p->hi_img_host.assign((size_t)L * E, nullptr);
    const bool ssd = ssd_path != nullptr;
    if (ssd) {
        // f-4: every HIGH image in one file (written below), a pinned LRU cache of ssd_slots images in front
        p->ssd_fd = open(ssd_path, O_RDWR | O_CREAT | O_TRUNC, 0600);
        if (p->ssd_fd < 0) { dx_set_error("cannot create the SSD tier file %s", ssd_path); return fail(DX_ERR_INVALID_ARG); }
        p->ssd_path = ssd_path;
        p->ssd_slots = ssd_slots;
        ce = cudaHostAlloc((void**)&p->ssd_cache, (size_t)ssd_slots * p->img_bytes, cudaHostAllocDefault);
        if (ce != cudaSuccess) { dx_set_error("cudaHostAlloc SSD-tier DRAM cache: %s", cudaGetErrorString(ce)); return fail(DX_ERR_OOM); }
        p->cache_slot_of.assign((size_t)L * E, -1);
        p->cache_owner.assign(ssd_slots, -1);
        p->cache_used.assign(ssd_slots, 0);
        p->cache_ev.resize(ssd_slots);
        for (int i = 0; i < ssd_slots; ++i) cudaEventCreateWithFlags(&p->cache_ev[i], cudaEventDisableTiming);
    } else if (cfg->high_bits < 16) {
        ce = cudaHostAlloc((void**)&p->hi_cache, (size_t)L * E * p->hi.bytes, cudaHostAllocMapped | cudaHostAllocPortable);
        if (ce != cudaSuccess) { dx_set_error("cudaHostAlloc HIGH cache: %s", cudaGetErrorString(ce)); return fail(DX_ERR_OOM); }
    }
    std::vector<const uint8_t*> img_dev((size_t)L * E, nullptr);
    for (int l = 0; l < L; ++l)
        for (int e = 0; e < E; ++e) {
            const void* m = master[(size_t)l * E + e];
            if (!m) { dx_set_error("null master pointer (layer %d expert %d)", l, e); return fail(DX_ERR_INVALID_ARG); }
            const uint8_t* src_host;
            if (cfg->high_bits == 16) src_host = (const uint8_t*)m;
            else if (ssd) continue;                  // int HIGH images go to the file as they are quantised
            else src_host = p->hi_cache + ((size_t)l * E + e) * p->hi.bytes;
            cudaPointerAttributes at;
            ce = cudaPointerGetAttributes(&at, src_host);
            if (ce != cudaSuccess || at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) {
                cudaGetLastError();
                dx_set_error("master image of layer %d expert %d is not pinned/mapped host memory", l, e);
                return fail(DX_ERR_INVALID_ARG);
            }
            if (ssd) continue;                       // promotions read the file through the cache, not the masters
            p->hi_img_host[(size_t)l * E + e] = src_host;
            img_dev[(size_t)l * E + e] = (const uint8_t*)at.devicePointer;
        }
    DX_CUDA(cudaMemcpyAsync(p->hi_img_dev, img_dev.data(), img_dev.size() * sizeof(void*), cudaMemcpyHostToDevice, p->cs));

    // ---- controller initial state: warm-up layout, all LOW, expert e in LOW block e (R-P3)
    {
        std::vector<int32_t> tier(LE, 0), slot(LE), pend(LE, 0), own_lo(LO, -1), own_hi(LO, -1);
        std::vector<uint32_t> ver(LE, 0);
        std::vector<double> S(LE, 0.0);
        std::vector<i64> last(LE, DX_NEVER), at(LE, 0), tt(L, 0);
        std::vector<double> tau(L, INFINITY);
        std::vector<int32_t> clo(L, E), chi(L, 0), pn(L, 0);
        for (int l = 0; l < L; ++l)
            for (int e = 0; e < E; ++e) { slot[(size_t)l * E + e] = e; own_lo[(size_t)l * (E + s) + e] = e; }
        DX_CUDA(cudaMemcpyAsync(c.tier, tier.data(), LE * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.slot, slot.data(), LE * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.version, ver.data(), LE * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.S, S.data(), LE * 8, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemsetAsync(c.cnt, 0, LE * 4, p->cs));
        DX_CUDA(cudaMemsetAsync(c.mass, 0, LE * 8, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.last, last.data(), LE * 8, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.pend_dir, pend.data(), LE * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.pend_dst, pend.data(), LE * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.pend_at, at.data(), LE * 8, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.lo_owner, own_lo.data(), LO * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.hi_owner, own_hi.data(), LO * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.t, tt.data(), L * 8, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.tau, tau.data(), L * 8, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.cap_lo, clo.data(), L * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.cap_hi, chi.data(), L * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemcpyAsync(c.plan_n, pn.data(), L * 4, cudaMemcpyHostToDevice, p->cs));
        DX_CUDA(cudaMemsetAsync(p->err_flag, 0, 4, p->cs));
        DX_CUDA(cudaMemsetAsync(p->dev_err, 0, 4, p->cs));
        DX_CUDA(cudaMemsetAsync(p->gemm_sched, 0, 48, p->cs));
        DX_CUDA(cudaMemsetAsync(p->dn_done, 0, ((size_t)p->E_loc + 64) * 4, p->cs));
        DX_CUDA(cudaMemsetAsync(w.stats, 0, 4 * 8, p->cs));
        DX_CUDA(cudaMemsetAsync(w.done, 0, 4, p->cs));
        DX_CUDA(cudaMemsetAsync(w.gbar, 0, 8, p->cs));
        if (p->ws_src.done) {                                // dispatch-side workspace (EP, loopback included)
            DX_CUDA(cudaMemsetAsync(p->ws_src.done, 0, 4, p->cs));
            DX_CUDA(cudaMemsetAsync(p->ws_src.gbar, 0, 8, p->cs));
        }
        DX_CUDA(cudaMemsetAsync(c.tstats, 0, 16, p->cs));
        if (p->L > 1) DX_CUDA(cudaMemsetAsync(p->corr, 0, (size_t)(p->L - 1) * p->E_loc * p->E_loc * 4, p->cs));
        DX_CUDA(cudaStreamSynchronize(p->cs));
    }
    for (int ti = 0; ti < 2; ++ti) {
        const SlotLayout& Ls = ti ? p->hi : p->lo;
        p->wbytes[ti][0] = phase_bytes(Ls, p->H, p->I, p->g, 2);
        p->wbytes[ti][1] = phase_bytes(Ls, p->H, p->I, p->g, 1);
    }

    // ---- initial images: LOW block e of every expert (and the HIGH image cache if quantised)
    const size_t mbytes = (size_t)3 * p->I * p->H * 2;
    SlotLayout bf = dx_slot_layout(p->H, p->I, p->g, 16);
    for (int l = 0; l < L; ++l)
        for (int e = 0; e < E; ++e) {
            DX_CUDA(cudaMemcpyAsync(stage_master, master[(size_t)l * E + e], mbytes, cudaMemcpyHostToDevice, p->cs));
            uint8_t* low = p->weights + (size_t)l * p->layer_bytes + (size_t)e * p->lo.bytes;
            if (cfg->high_bits == 16) {
                launch_quantize_slot(stage_master, bf, low, p->lo, p->H, p->I, p->g, p->cs);
                if (ssd) {
                    dx_status st2 = ssd_write(p, (size_t)l * E + e, master[(size_t)l * E + e]);
                    if (st2 != DX_OK) return fail(st2);
                }
            } else {
                launch_quantize_slot(stage_master, bf, stage_high, p->hi, p->H, p->I, p->g, p->cs);
                uint8_t* dst = ssd ? p->ssd_cache : p->hi_cache + ((size_t)l * E + e) * p->hi.bytes;
                DX_CUDA(cudaMemcpyAsync(dst, stage_high, p->hi.bytes, cudaMemcpyDeviceToHost, p->cs));
                launch_quantize_slot(stage_high, p->hi, low, p->lo, p->H, p->I, p->g, p->cs);
                if (ssd) {
                    DX_CUDA(cudaStreamSynchronize(p->cs));
                    dx_status st2 = ssd_write(p, (size_t)l * E + e, p->ssd_cache);
                    if (st2 != DX_OK) return fail(st2);
                }
            }
            p->launches += cfg->high_bits == 16 ? 3 : 6;
        }
    for (int l = 0; l < L && cfg->n_shared; ++l) {           // f-3: shared experts, HIGH tier, their own block
        const void* m = master[(size_t)L * E + l];
        if (!m) { dx_set_error("null shared-expert master pointer (layer %d)", l); return fail(DX_ERR_INVALID_ARG); }
        uint8_t* blk = p->weights + (size_t)l * p->layer_bytes + p->hi_base + (size_t)p->shared_slot * p->hi.bytes;
        DX_CUDA(cudaMemcpyAsync(stage_master, m, mbytes, cudaMemcpyHostToDevice, p->cs));
        if (cfg->high_bits == 16) DX_CUDA(cudaMemcpyAsync(blk, stage_master, mbytes, cudaMemcpyDeviceToDevice, p->cs));
        else launch_quantize_slot(stage_master, bf, blk, p->hi, p->H, p->I, p->g, p->cs);
    }
    DX_CUDA(cudaStreamSynchronize(p->cs));
    DX_CUDA(cudaGetLastError());
    if (ssd) {
        // the file is the SSD tier from here on: flush it and drop it from the page cache (reads are O_DIRECT when
        // the image size allows, so a promotion that misses the DRAM cache really reads the device)
        fsync(p->ssd_fd);
        posix_fadvise(p->ssd_fd, 0, 0, POSIX_FADV_DONTNEED);
        const int fd2 = open(ssd_path, O_RDONLY | O_DIRECT);
        if (fd2 >= 0 && p->img_bytes % 4096 == 0) { close(p->ssd_fd); p->ssd_fd = fd2; p->ssd_direct = true; }
        else if (fd2 >= 0) close(fd2);
    }
    {
        // the transfer thread: issues the SSD tier's reads and copies off the forward-issuing host thread.  For DRAM
        // pools it is opt-in (DX_XFER_THREAD=1): measured, it did not lower the exposed switch time and the hand-over
        // at publication cost the end-to-end loop (host copy + sync every step) ~6 %
        static const bool xt = [] { const char* e = getenv("DX_XFER_THREAD"); return e && atoi(e) != 0; }();
        if (ssd || (xt && !nccl_id && !ep_group)) {
            cudaGetDevice(&p->device);
            p->io_pending.assign(L, 0);
            p->io_thread = std::thread(io_worker, p);
        }
    }

    dx_info& inf = p->info;
    inf.n_hot = (int)n_hot;
    inf.experts_local = E;
    inf.cap_hi = cap_hi;
    inf.cap_lo = cap_lo;
    inf.slot_bytes_hi = p->hi.bytes;
    inf.slot_bytes_lo = p->lo.bytes;
    inf.layer_budget = M;
    inf.layer_bytes = p->layer_bytes;
    inf.arena_bytes = (i64)total;
    const i64 n3 = (i64)3 * p->I * p->H;
    inf.export_bytes_hi = cfg->high_bits == 16 ? n3 * 2 : n3 + n3 / p->g * 3;
    inf.export_bytes_lo = n3 + n3 / p->g * 3;
    gemm_trap_init();
    st = build_maps(p);
    if (st != DX_OK) return fail(st);
    *out = p;
    return DX_OK;
}

extern "C" dx_status dx_set_ffn_path(dx_pool p, int32_t path) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    DX_CHECK(path == 0 || p->cfg.n_shared == 0, DX_ERR_INVALID_ARG, "the shared expert runs on the tcgen05 path only");
    DX_CHECK(path == 0 || !(p->comm || p->ep_group), DX_ERR_INVALID_ARG,
             "the in-library EP layer (deduplicated rows) runs on the tcgen05 path only");
    DX_CHECK(path == 0 || path == 1, DX_ERR_INVALID_ARG, "path must be 0 (tcgen05) or 1 (mma.sync)");
    p->ffn_path = path;
    return DX_OK;
}

extern "C" dx_status dx_pool_create(const dx_config* cfg, const void* const* master, void* compute_stream,
                                    void* side_stream, dx_pool* out) {
    return pool_create(cfg, master, compute_stream, side_stream, nullptr, out);
}

extern "C" dx_status dx_pool_create_ep(const dx_config* cfg, const void* const* master, void* compute_stream,
                                       void* side_stream, const void* nccl_id, dx_pool* out) {
    // nccl_id NULL: a member of a local pool group (several ranks' pools in one process, dx_moe_step_group)
    return pool_create(cfg, master, compute_stream, side_stream, nccl_id, out, nullptr, 0, nccl_id == nullptr);
}

extern "C" dx_status dx_pool_create_ssd(const dx_config* cfg, const void* const* master, void* compute_stream,
                                        void* side_stream, const char* ssd_path, int32_t dram_cache_images, dx_pool* out) {
    DX_CHECK(ssd_path && *ssd_path, DX_ERR_INVALID_ARG, "null SSD tier path");
    DX_CHECK(dram_cache_images >= 1, DX_ERR_INVALID_ARG, "the DRAM cache needs at least one image slot");
    DX_CHECK(cfg && cfg->ep_size == 1, DX_ERR_INVALID_ARG, "the SSD tier is for ep_size == 1 pools");
    return pool_create(cfg, master, compute_stream, side_stream, nullptr, out, ssd_path, dram_cache_images);
}

extern "C" dx_status dx_get_unique_id(void* id128) {
    DX_CHECK(id128, DX_ERR_INVALID_ARG, "null id");
    return ep_nccl_unique_id(id128);
}

extern "C" dx_status dx_pool_destroy(dx_pool p) {
    if (!p) return DX_OK;
    if (p->io_thread.joinable()) {
        {
            std::lock_guard<std::mutex> lk(p->io_mu);
            p->io_stop = true;
        }
        p->io_cv.notify_all();
        p->io_thread.join();
    }
    if (p->cs) cudaStreamSynchronize(p->cs);
    if (p->ss) cudaStreamSynchronize(p->ss);
    if (p->comm) ep_nccl_destroy(p->comm);
    if (p->ep_pairs_host) cudaFreeHost(p->ep_pairs_host);
    for (auto ev : p->ev_planh) cudaEventDestroy(ev);
    for (auto ev : p->ev_plandone) cudaEventDestroy(ev);
    for (auto ev : p->ev_pf) cudaEventDestroy(ev);
    for (auto ev : p->cache_ev) cudaEventDestroy(ev);
    if (p->ssd_cache) cudaFreeHost(p->ssd_cache);
    if (p->ssd_fd >= 0) { close(p->ssd_fd); unlink(p->ssd_path.c_str()); }
    if (p->pf_host) cudaFreeHost(p->pf_host);
    if (p->pf_n_host) cudaFreeHost(p->pf_n_host);
    if (p->ss2) { cudaStreamSynchronize(p->ss2); cudaStreamDestroy(p->ss2); }
    if (p->ev_dem) cudaEventDestroy(p->ev_dem);
    for (auto ev : p->prof_copy_ev) cudaEventDestroy(ev);
    if (p->plan_host) cudaFreeHost(p->plan_host);
    if (p->plan_n_host) cudaFreeHost(p->plan_n_host);
    for (auto ev : p->ev_side) cudaEventDestroy(ev);
    if (p->ev_plan) cudaEventDestroy(p->ev_plan);
    if (p->own_ss && p->ss) cudaStreamDestroy(p->ss);
    for (auto ev : p->prof_ev) cudaEventDestroy(ev);
    for (auto ev : p->prof_free) cudaEventDestroy(ev);
    if (p->hi_cache) cudaFreeHost(p->hi_cache);
    if (p->arena) cudaFree(p->arena);
    delete p;
    return DX_OK;
}

extern "C" dx_status dx_set_prefetch(dx_pool p, int32_t fanout, int32_t lead) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    DX_CHECK(fanout >= 0 && fanout <= 8, DX_ERR_INVALID_ARG, "fanout %d outside [0, 8]", (int)fanout);
    DX_CHECK(fanout == 0 || (lead >= 1 && lead <= p->cfg.period - p->cfg.publish_lag), DX_ERR_INVALID_ARG,
             "lead %d outside [1, Tp - L = %d]", (int)lead, p->cfg.period - p->cfg.publish_lag);
    DX_CHECK(fanout == 0 || (p->cfg.ep_size == 1 && !p->comm), DX_ERR_INVALID_ARG,
             "prefetch needs the whole stack on one GPU (ep_size 1)");
    p->pf_f = fanout;
    p->pf_lead = lead;
    p->T_last[0] = p->T_last[1] = -1;
    return DX_OK;
}

extern "C" dx_status dx_get_corr(dx_pool p, int32_t layer, uint32_t* host_out) {
    DX_CHECK(p && host_out, DX_ERR_INVALID_ARG, "null pool/out");
    DX_CHECK(layer >= 0 && layer + 1 < p->L, DX_ERR_RANGE, "layer pair (%d, %d) outside the stack", (int)layer,
             (int)layer + 1);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    DX_CUDA(cudaMemcpy(host_out, p->corr + (size_t)layer * p->E_loc * p->E_loc, (size_t)p->E_loc * p->E_loc * 4,
                       cudaMemcpyDeviceToHost));
    return DX_OK;
}

extern "C" dx_status dx_get_prefetch(dx_pool p, int32_t layer, int32_t* experts, int32_t* blocks, int32_t* n) {
    DX_CHECK(p && experts && blocks && n, DX_ERR_INVALID_ARG, "null argument");
    DX_CHECK(layer >= 0 && layer < p->L, DX_ERR_RANGE, "layer %d out of range", (int)layer);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    *n = 0;
    for (const int2& sg : p->staged[layer]) { experts[*n] = sg.x; blocks[*n] = sg.y; ++*n; }
    if (*n == 0 && p->pf_pending[layer]) {          // made but not issued yet: report the candidates themselves
        for (int i = 0; i < p->pf_n_host[layer]; ++i) {
            experts[i] = p->pf_host[(size_t)layer * 8 + i].x;
            blocks[i] = p->pf_host[(size_t)layer * 8 + i].y;
        }
        *n = p->pf_n_host[layer];
    }
    return DX_OK;
}

extern "C" dx_status dx_set_teleport(dx_pool p, int32_t on) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    p->teleport = on != 0;
    return DX_OK;
}

extern "C" dx_status dx_pool_info(dx_pool p, dx_info* out) {
    DX_CHECK(p && out, DX_ERR_INVALID_ARG, "null pool/out");
    *out = p->info;
    return DX_OK;
}

extern "C" int64_t dx_kernel_launches(dx_pool p) { return p ? p->launches : 0; }

extern "C" dx_status dx_profile_enable(dx_pool p, int32_t enable) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    p->profiling = enable != 0;
    p->prof_every = enable > 1 ? enable : 1;
    p->prof_ctr = 0;
    return DX_OK;
}

extern "C" dx_status dx_profile_read(dx_pool p, dx_profile_t* out) {
    {
        dx_status st = io_wait(p, -1);                      // SSD tier: every hand-over recorded its events
        if (st != DX_OK) return st;
    }
    DX_CHECK(p && out, DX_ERR_INVALID_ARG, "null pool/out");
    DX_CUDA(cudaStreamSynchronize(p->cs));
    DX_CUDA(cudaStreamSynchronize(p->ss));
    memset(out, 0, sizeof(*out));
    for (size_t i = 0; i + 3 < p->prof_ev.size(); i += 4) {
        float a = 0, b = 0, c = 0, d = 0;
        DX_CUDA(cudaEventElapsedTime(&a, p->prof_ev[i], p->prof_ev[i + 3]));
        DX_CUDA(cudaEventElapsedTime(&b, p->prof_ev[i + 1], p->prof_ev[i + 2]));
        DX_CUDA(cudaEventElapsedTime(&c, p->prof_ev[i + 2], p->prof_ev[i + 3]));
        DX_CUDA(cudaEventElapsedTime(&d, p->prof_ev[i], p->prof_ev[i + 1]));
        out->fwd_ms += a;
        out->ffn_ms[0] += b;
        out->ffn_ms[1] += c;
        out->route_ms += d;
    }
    for (size_t i = 0; i + 1 < p->prof_wait_ev.size(); i += 2) {
        float a = 0;
        DX_CUDA(cudaEventElapsedTime(&a, p->prof_wait_ev[i], p->prof_wait_ev[i + 1]));
        out->exposed_ms += a;
        out->publishes += 1;
    }
    for (size_t i = 0; i + 1 < p->prof_xfer_ev.size(); i += 2) {
        float a = 0;
        DX_CUDA(cudaEventElapsedTime(&a, p->prof_xfer_ev[i], p->prof_xfer_ev[i + 1]));
        out->xfer_ms += a;
        out->xfer_max_ms = a > out->xfer_max_ms ? a : out->xfer_max_ms;
        out->plans += 1;
    }
    out->ssd_reads = (int64_t)p->ssd_reads;
    out->ssd_bytes = p->ssd_bytes;
    out->ssd_read_ms = p->ssd_read_ms;
    out->dram_cache_hits = (int64_t)p->cache_hits;
    p->ssd_reads = p->ssd_bytes = p->cache_hits = 0;
    p->ssd_read_ms = 0.0;
    out->prefetch_issued = (int64_t)p->pf_issued;
    out->prefetch_hits = (int64_t)p->pf_hits;
    p->pf_issued = p->pf_hits = 0;
    for (size_t i = 0; i + 1 < p->prof_copy_ev.size(); i += 2) {
        float a = 0;
        DX_CUDA(cudaEventElapsedTime(&a, p->prof_copy_ev[i], p->prof_copy_ev[i + 1]));
        out->copy_ms += a;
        out->copy_bytes += p->prof_copy_bytes[i / 2];
    }
    for (size_t i = 0; i < p->prof_copy_ev.size(); i += 2) p->prof_free.push_back(p->prof_copy_ev[i + 1]);
    p->prof_copy_ev.clear();
    p->prof_copy_bytes.clear();
    for (auto e : p->prof_ev) p->prof_free.push_back(e);
    for (auto e : p->prof_wait_ev) p->prof_free.push_back(e);
    for (auto e : p->prof_xfer_ev) p->prof_free.push_back(e);
    p->prof_ev.clear();
    p->prof_wait_ev.clear();
    p->prof_xfer_ev.clear();
    out->forwards = p->prof_fwd;
    p->prof_fwd = 0;
    out->ffn_fused = p->prof_fused;
    p->prof_fused = 0;
    u64 st[4];
    DX_CUDA(cudaMemcpy(st, p->ws.stats, sizeof(st), cudaMemcpyDeviceToHost));
    DX_CUDA(cudaMemset(p->ws.stats, 0, sizeof(st)));
    out->weight_bytes[0] = st[0];
    out->weight_bytes[1] = st[1];
    out->active_experts = st[2];
    u64 ts[2];
    DX_CUDA(cudaMemcpy(ts, p->ctrl.tstats, sizeof(ts), cudaMemcpyDeviceToHost));
    DX_CUDA(cudaMemset(p->ctrl.tstats, 0, sizeof(ts)));
    out->promotions = (int64_t)ts[0];
    out->demotions = (int64_t)ts[1];
    return DX_OK;
}

static dx_status expert_ffn(dx_pool p, int layer, const RouteWs& ws, const void* x, int T, int k, void* y,
                            cudaEvent_t* ev, bool fuse_fold = false, int m_max = -1);
static bool prof_begin(dx_pool p, cudaEvent_t* ev);
static dx_status fold(dx_pool p, int layer);
static dx_status fold_prepare(dx_pool p, int layer, FoldReq* req);

#define CHECK_LAYER(p, layer)                                                                          \
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");                                                      \
    DX_CHECK((layer) >= 0 && (layer) < (p)->L, DX_ERR_RANGE, "layer %d out of range [0,%d)", (int)(layer), (p)->L)

// a1-a5: routing of T tokens over this pool's experts into `ws` (+ the x gather for the tcgen05 path).
// Decode batches (T*k <= 512): one fused multi-CTA launch; larger batches: router, top-k/counters/scan,
// placement.
static void route_tokens(dx_pool p, int layer, const void* x, int T, const void* router_w, const float* router_bias,
                         const float* logits, RouteWs& ws) {
    const size_t base = (size_t)layer * p->E_loc;
    __nv_bfloat16* Xp = p->ffn_path == 1 ? nullptr : p->Xp;
    if (route_dec_ok(T, p->E, p->k)) {
        launch_route_dec((const __nv_bfloat16*)x, (const __nv_bfloat16*)router_w, router_bias, router_w ? nullptr : logits,
                         T, p->E, p->k, p->H, p->e_lo, ws, p->ctrl.cnt + base, p->ctrl.mass + base, p->ctrl.tier + base,
                         p->wbytes, Xp, p->cs);
        p->launches += 1;
        return;
    }
    const float* lg = logits;
    if (router_w) {
        launch_router((const __nv_bfloat16*)x, (const __nv_bfloat16*)router_w, router_bias, T, p->E, p->H, ws.logits,
                      p->cs);
        lg = ws.logits;
        p->launches += 1;
    }
    launch_route(lg, T, p->E, p->k, p->e_lo, ws, p->ctrl.cnt + base, p->ctrl.mass + base, p->ctrl.tier + base,
                 p->wbytes, p->cs);
    launch_place(T, p->E, p->k, ws, (const __nv_bfloat16*)x, p->H, Xp, p->cs);
    p->launches += 3;
}

static dx_status ep_forward(dx_pool p, int layer, const void* x, int T, const void* router_w, const float* router_bias,
                            const float* logits, void* y, int32_t* topk_idx, float* topk_gate, bool fuse_fold);
static dx_status poll_transfers(dx_pool p, int wait_layer = -1);

// f-1 after layer `layer`'s routing (idx [T][k] on the compute stream): the correlation counts of the pair
// (layer - 1, layer) when the previous layer routed the same batch, this routing kept for the next layer, and --
// `pf_lead` steps before layer + 1's next plan -- that layer's prefetch candidates, read back like a plan.
static dx_status prefetch_hooks(dx_pool p, int layer, const int32_t* idx, int T) {
    const int k = p->k, E = p->E_loc, par = layer & 1;
    const bool upd = layer >= 1 && p->T_last[par ^ 1] == T;
    launch_corr(upd ? p->idx_last + (size_t)(par ^ 1) * p->cfg.max_tokens * k : nullptr, idx, T, k, E,
                upd ? p->corr + (size_t)(layer - 1) * E * E : nullptr, p->idx_last + (size_t)par * p->cfg.max_tokens * k,
                p->cs);
    p->launches += 1;
    p->T_last[par] = T;
    const int nl = layer + 1;
    if (nl >= p->L || !p->finalized[nl] || p->pf_pending[nl] || p->publish_at[nl] >= 0) return DX_OK;
    const i64 t = p->t[nl];                                   // layer nl's step count: this batch's step
    if (t <= p->cfg.warmup_steps || (t + p->pf_lead) % p->cfg.period != 0) return DX_OK;
    launch_prefetch(p->ctrl, nl, p->corr + (size_t)layer * E * E, idx, T, k, p->pf_f, p->pf_dev + (size_t)nl * 8,
                    p->pf_n_dev + nl, p->cs);
    DX_CUDA(cudaMemcpyAsync(p->pf_host + (size_t)nl * 8, p->pf_dev + (size_t)nl * 8, 8 * sizeof(int4),
                            cudaMemcpyDeviceToHost, p->cs));
    DX_CUDA(cudaMemcpyAsync(p->pf_n_host + nl, p->pf_n_dev + nl, sizeof(int32_t), cudaMemcpyDeviceToHost, p->cs));
    DX_CUDA(cudaEventRecord(p->ev_pf[nl], p->cs));
    p->pf_pending[nl] = 1;
    p->n_pending += 1;
    p->launches += 1;
    return DX_OK;
}

// the staged copies of layer `layer`'s prefetch candidates (H2D on the copy engine into free HIGH blocks)
static dx_status issue_prefetch(dx_pool p, int layer) {
    const size_t bytes = p->hi.bits == 16 ? (size_t)3 * p->I * p->H * 2 : (size_t)p->hi.bytes;
    uint8_t* hi_region = p->weights + (size_t)layer * p->layer_bytes + p->hi_base;
    const int n = p->pf_n_host[layer];
    p->staged[layer].clear();
    for (int i = 0; i < n; ++i) {
        const int4 c = p->pf_host[(size_t)layer * 8 + i];
        dx_status rc = copy_high_image(p, (size_t)layer * p->E_loc + c.x, hi_region + (size_t)c.y * p->hi.bytes, p->ss);
        if (rc != DX_OK) return rc;
        p->staged[layer].push_back(make_int2(c.x, c.y));
    }
    p->pf_issued += (u64)n;
    p->pf_pending[layer] = 0;
    p->n_pending -= 1;
    return DX_OK;
}

static dx_status forward_impl(dx_pool p, int32_t layer, const void* x, int32_t T, const void* router_w,
                              const float* router_bias, const float* logits, void* y, int32_t* topk_idx,
                              float* topk_gate, bool fuse_fold) {
    CHECK_LAYER(p, layer);
    DX_CHECK(T >= 0 && T <= p->cfg.max_tokens, DX_ERR_RANGE, "T=%d outside [0, max_tokens=%d]", T, p->cfg.max_tokens);
    DX_CHECK(T == 0 || (x && y), DX_ERR_INVALID_ARG, "null x/y");
    DX_CHECK(T == 0 || (router_w != nullptr) != (logits != nullptr), DX_ERR_INVALID_ARG,
             "exactly one of router_w (router mode) and logits (trace mode) must be given");
    {
        dx_status st = poll_transfers(p);
        if (st != DX_OK) return st;
    }
    if (p->comm) return ep_forward(p, layer, x, T, router_w, router_bias, logits, y, topk_idx, topk_gate, fuse_fold);
    DX_CHECK(p->cfg.ep_size == 1, DX_ERR_INVALID_ARG,
             "ep_size > 1 without a communicator (dx_pool_create_ep): use dx_ep_dispatch / dx_moe_forward_routed / "
             "dx_ep_combine");
    if (T == 0) return fuse_fold ? fold(p, layer) : DX_OK;
    cudaEvent_t ev[4];
    const bool sampled = prof_begin(p, ev);
    RouteWs ws = p->ws;
    if (p->profiling && !sampled) ws.stats = nullptr;   // byte counters follow the sampled forwards
    if (topk_idx) ws.idx = topk_idx;
    if (topk_gate) ws.gate = topk_gate;
    p->last_logits_router = router_w != nullptr;
    p->last_T = T;
    route_tokens(p, layer, x, T, router_w, router_bias, logits, ws);
    if (p->pf_f > 0) {
        dx_status st = prefetch_hooks(p, layer, ws.idx, T);
        if (st != DX_OK) return st;
    }
    if (p->cfg.n_shared) {                                    // f-3: the shared expert's rows after the routed ones
        launch_shared_rows(ws, T, p->k, p->E_loc, p->H, (const __nv_bfloat16*)x, p->ffn_path == 1 ? nullptr : p->Xp,
                           p->wbytes[1][0], p->wbytes[1][1], p->cs);
        p->launches += 1;
    }
    p->pend_tokens[layer] += (u64)T;
    return expert_ffn(p, layer, ws, x, T, p->k, y, ev, fuse_fold);
}

extern "C" dx_status dx_moe_forward(dx_pool p, int32_t layer, const void* x, int32_t T, const void* router_w,
                                    const float* router_bias, const float* logits, void* y, int32_t* topk_idx,
                                    float* topk_gate) {
    return forward_impl(p, layer, x, T, router_w, router_bias, logits, y, topk_idx, topk_gate, false);
}

extern "C" dx_status dx_moe_step(dx_pool p, int32_t layer, const void* x, int32_t T, const void* router_w,
                                 const float* router_bias, const float* logits, void* y, int32_t* topk_idx,
                                 float* topk_gate) {
    dx_status st = forward_impl(p, layer, x, T, router_w, router_bias, logits, y, topk_idx, topk_gate, true);
    if (st != DX_OK) return st;
    return dx_plan_precision(p, layer, nullptr);
}

extern "C" dx_status dx_moe_step_layers(dx_pool p, int32_t layer0, int32_t n_layers, const void* const* x, int32_t T,
                                        const void* const* router_w, const float* const* router_bias,
                                        const float* const* logits, void* const* y) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    DX_CHECK(n_layers >= 0 && layer0 >= 0 && layer0 + n_layers <= p->L, DX_ERR_RANGE, "layers [%d, %d) outside [0, %d)",
             (int)layer0, (int)(layer0 + n_layers), p->L);
    DX_CHECK(x && y && (router_w || logits), DX_ERR_INVALID_ARG, "null pointer array");
    for (int i = 0; i < n_layers; ++i) {
        dx_status st = dx_moe_step(p, layer0 + i, x[i], T, router_w ? router_w[i] : nullptr,
                                   router_bias ? router_bias[i] : nullptr, logits ? logits[i] : nullptr, y[i], nullptr,
                                   nullptr);
        if (st != DX_OK) return st;
    }
    return DX_OK;
}

extern "C" dx_status dx_get_logits(dx_pool p, float* host_out, int64_t cap) {
    DX_CHECK(p && host_out, DX_ERR_INVALID_ARG, "null pool/out");
    DX_CHECK(p->last_logits_router, DX_ERR_NOT_READY, "the last forward was not in router mode");
    const int64_t n = (int64_t)p->last_T * p->E;
    DX_CHECK(cap >= n, DX_ERR_INVALID_ARG, "output too small (%lld < %lld)", (long long)cap, (long long)n);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    DX_CUDA(cudaMemcpy(host_out, p->ws.logits, n * 4, cudaMemcpyDeviceToHost));
    return DX_OK;
}

// a6-a8 on rows already routed and placed in `ws`: grouped expert GEMMs over the slot pool, then the
// weighted combine of k rows per token into y (k = 1: the rows themselves, EP owner side).
// m_max: an upper bound on any expert's row count (-1: T, as for top-k routing of T tokens)
static dx_status expert_ffn(dx_pool p, int layer, const RouteWs& ws, const void* x, int T, int k, void* y,
                            cudaEvent_t* ev, bool fuse_fold, int m_max) {
    const size_t base = (size_t)layer * p->E_loc;
    const int E = p->E_loc;
    ExpertArgs a;
    a.arena_layer = p->weights + (size_t)layer * p->layer_bytes;
    a.tier = p->ctrl.tier + base;
    a.slot = p->ctrl.slot + base;
    a.hi_base = p->hi_base;
    a.hi = p->hi;
    a.lo = p->lo;
    a.H = p->H; a.I = p->I; a.g = p->g; a.k = k;
    if (ev[1]) DX_CUDA(cudaEventRecord(ev[1], p->cs));
    const int ns = k == p->k ? p->cfg.n_shared : 0;            // the owner-side (k = 1) EP path has no shared rows
    int ffn_launches = 2;                                       // kernels launched for a6/a7 (counted below)
    const int max_act = (T * k < E ? T * k : E) + ns;
    if (p->ffn_path == 1) {
        launch_expert_ffn(a, (const __nv_bfloat16*)x, ws.gate, ws, T, E, p->act, p->Y, p->cs, ev[2]);
    } else {
        // tcgen05 grouped GEMMs (k_gemm.cu) over the rows placed in Xp: gate/up + SwiGLU, then down.
        // m_e <= T for top-k routing; the owner side (k = 1) sees m_e <= T rows as well.
        const bool dec = gemm_decode_cfg(m_max >= 0 ? m_max : T);
        {
        GemmArgs ga;
        ga.layer = a.arena_layer; ga.hi_base = p->hi_base; ga.hi = p->hi; ga.lo = p->lo;
        ga.tier = a.tier; ga.slot = a.slot; ga.off = ws.off; ga.act_e = ws.act_e; ga.n_act = ws.n_act;
        ga.perm = ws.perm; ga.gate = ws.gate; ga.H = p->H; ga.I = p->I; ga.g = p->g; ga.k = k;
        ga.act = p->act; ga.Y = p->Y; ga.sched = p->gemm_sched;
        ga.E_loc = E; ga.shared_slot = p->shared_slot;
        static const int dbg = [] { const char* s = getenv("DX_GEMM_DBG"); return s ? atoi(s) : 0; }();
        ga.dbg = dbg;
        // prefill with a bf16 HIGH tier: those experts' items run as 128 x 256 tiles in k_wide, the rest in k_gemm
        const bool wide = !dec && p->hi.bits == 16 && wide_enabled();
        ga.skip_bf16 = wide ? 1 : 0;
        ga.dn_done = p->dn_done;
        GemmMaps gm = p->gmaps[layer];
        for (int i = 0; i < 4; ++i) gm.xb[i] = p->xb0[i];
        for (int i = 0; i < 3; ++i) gm.xk[i] = p->xk0[i];
        gm.xw = p->xw0;
        gm.xb192 = p->xp0;
        static const bool fuse_on = [] { const char* e = getenv("DX_FUSE"); return !e || atoi(e) != 0; }();
        if (dec && fuse_on) {
            // decode: gate/up + SwiGLU and down + gate scaling in ONE launch (down items wait per expert)
            for (int i = 0; i < 4; ++i) gm.xb1[i] = p->xb1[i];
            for (int i = 0; i < 3; ++i) gm.xk1[i] = p->xk1[i];
            launch_gemm(2, true, gm, ga, max_act * (p->I / 64 + (p->H + 127) / 128), p->cs);
            ffn_launches = 1;
            if (ev[2]) {
                DX_CUDA(cudaEventRecord(ev[2], p->cs));
                ++p->prof_fused;
            }
        } else {
        if (wide) launch_wide(0, gm, ga, max_act * (p->I / 64), p->cs);
        if (wide) ffn_launches = 4;
        launch_gemm(0, dec, gm, ga, max_act * (p->I / 64), p->cs);
        if (ev[2]) DX_CUDA(cudaEventRecord(ev[2], p->cs));
        for (int i = 0; i < 4; ++i) gm.xb[i] = p->xb1[i];
        for (int i = 0; i < 3; ++i) gm.xk[i] = p->xk1[i];
        gm.xw = p->xw1;
        gm.xb192 = p->xp1;
        if (wide) launch_wide(1, gm, ga, max_act * ((p->H + 127) / 128), p->cs);
        launch_gemm(1, dec, gm, ga, max_act * ((p->H + 127) / 128), p->cs);
        }
        }
    }
    if (ev[3]) DX_CUDA(cudaEventRecord(ev[3], p->cs));
    if (fuse_fold) {
        // a8 + a10 + a14 in one launch: the fold block runs after the down GEMM (griddepcontrol.wait)
        FoldReq req;
        dx_status st = fold_prepare(p, layer, &req);
        if (st != DX_OK) return st;
        launch_combine(p->Y, T, k, p->H, (__nv_bfloat16*)y, p->cs, nullptr, &p->ctrl, &req, ns ? T * k : -1);
    } else {
        launch_combine(p->Y, T, k, p->H, (__nv_bfloat16*)y, p->cs, nullptr, nullptr, nullptr, ns ? T * k : -1);
    }
    p->launches += ffn_launches + 1;                            // + the combine
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "launch failed: %s", cudaGetErrorString(ce));
    static const bool log_bytes = getenv("DX_LOG_BYTES") != nullptr;
    if (log_bytes && ws.stats) {   // evidence runs (ncu traffic pairing): this forward's algorithmic bytes per phase
        static u64 prev[2] = {0, 0};
        u64 st[2];
        DX_CUDA(cudaStreamSynchronize(p->cs));
        DX_CUDA(cudaMemcpy(st, ws.stats, sizeof(st), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 2; ++i) if (st[i] < prev[i]) prev[i] = 0;      // counters were reset in between
        fprintf(stderr, "DX_LOG_BYTES layer %d T %d gateup %llu down %llu\n", layer, T,
                (unsigned long long)(st[0] - prev[0]), (unsigned long long)(st[1] - prev[1]));
        prev[0] = st[0];
        prev[1] = st[1];
    }
    return DX_OK;
}

static bool prof_begin(dx_pool p, cudaEvent_t* ev) {
    ev[0] = ev[1] = ev[2] = ev[3] = nullptr;
    if (!p->profiling) return false;
    if (p->prof_ctr++ % p->prof_every != 0) return false;      // not a sampled forward
    for (int i = 0; i < 4; ++i) {
        ev[i] = prof_event(p);
        p->prof_ev.push_back(ev[i]);
    }
    cudaEventRecord(ev[0], p->cs);
    p->prof_fwd += 1;
    return true;
}

// ---------------------------------------------------------------- expert parallelism (a15)
static dx_status ep_dispatch_impl(dx_pool p, int32_t layer, const void* x, int32_t T, const void* router_w,
                                  const float* router_bias, const float* logits, void* send_rows, void* send_meta,
                                  int32_t* send_counts, int32_t* send_pairs, int32_t* topk_idx, float* topk_gate) {
    CHECK_LAYER(p, layer);
    DX_CHECK(p->cfg.ep_size > 1 || p->comm, DX_ERR_INVALID_ARG, "dx_ep_dispatch needs ep_size > 1 (use dx_moe_forward)");
    DX_CHECK(T >= 0 && T <= p->cfg.max_tokens, DX_ERR_RANGE, "T=%d outside [0, max_tokens]", T);
    DX_CHECK(T == 0 || (router_w != nullptr) != (logits != nullptr), DX_ERR_INVALID_ARG, "exactly one of router_w / logits");
    DX_CHECK(send_rows && send_meta && (send_counts || send_pairs) && (T == 0 || x), DX_ERR_INVALID_ARG, "null buffer");
    p->ep_T = T;
    if (T == 0) {
        if (send_counts) DX_CUDA(cudaMemsetAsync(send_counts, 0, sizeof(int32_t) * p->cfg.ep_size, p->cs));
        if (send_pairs) DX_CUDA(cudaMemsetAsync(send_pairs, 0, sizeof(int32_t) * 2 * p->cfg.ep_size, p->cs));
        return DX_OK;
    }
    RouteWs ws = p->ws_src;
    if (topk_idx) ws.idx = topk_idx;
    if (topk_gate) ws.gate = topk_gate;
    p->ws_src_live = ws;
    const float* lg = logits;
    if (router_w) {
        launch_router((const __nv_bfloat16*)x, (const __nv_bfloat16*)router_w, router_bias, T, p->E, p->H, ws.logits,
                      p->cs);
        lg = ws.logits;
        p->launches += 1;
    }
    const u64 nob[2][2] = {{0, 0}, {0, 0}};
    // top-k over the GLOBAL experts; no hotness here (owners count what they receive)
    launch_route(lg, T, p->E, p->k, 0, ws, nullptr, nullptr, nullptr, nob, p->cs);
    // rows sorted by global expert = grouped by owner rank: the placement IS the send buffer
    launch_place(T, p->E, p->k, ws, (const __nv_bfloat16*)x, p->H, (__nv_bfloat16*)send_rows, p->cs);
    launch_ep_meta(ws, T * p->k, p->E_loc, p->cfg.ep_size, (int2*)send_meta, send_counts, (int2*)send_pairs, T, p->cs);
    p->launches += 4;
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "dispatch launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

extern "C" dx_status dx_ep_dispatch(dx_pool p, int32_t layer, const void* x, int32_t T, const void* router_w,
                                    const float* router_bias, const float* logits, void* send_rows, void* send_meta,
                                    int32_t* send_counts, int32_t* topk_idx, float* topk_gate) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    DX_CHECK(send_counts, DX_ERR_INVALID_ARG, "null send_counts");
    return ep_dispatch_impl(p, layer, x, T, router_w, router_bias, logits, send_rows, send_meta, send_counts, nullptr,
                            topk_idx, topk_gate);
}

static dx_status routed_impl(dx_pool p, int32_t layer, const void* rows, int32_t R, const void* meta, void* y_rows,
                             int64_t tokens_global, const int32_t* rowmap = nullptr) {
    CHECK_LAYER(p, layer);
    DX_CHECK(R >= 0 && (size_t)R <= p->n_ent, DX_ERR_RANGE, "R=%d exceeds the workspace (%zu rows)", R, p->n_ent);
    DX_CHECK(tokens_global >= 0, DX_ERR_INVALID_ARG, "tokens_global < 0");
    p->pend_tokens[layer] += (u64)tokens_global;
    if (R == 0) return DX_OK;
    DX_CHECK(rows && meta && y_rows, DX_ERR_INVALID_ARG, "null buffer");
    cudaEvent_t ev[4];
    const bool sampled = prof_begin(p, ev);
    RouteWs ws = p->ws;
    if (p->profiling && !sampled) ws.stats = nullptr;   // byte counters follow the sampled forwards
    const size_t base = (size_t)layer * p->E_loc;
    // an out-of-range expert id in `meta` is routed to expert 0 with gate 0 (its output row is 0) and raises
    // the sticky device error that the next dx_sync reports as DX_ERR_RANGE
    launch_route_given((const int2*)meta, R, p->E_loc, ws, p->ctrl.cnt + base, p->ctrl.mass + base,
                       p->ctrl.tier + base, p->wbytes, p->dev_err, p->cs);
    launch_place(R, p->E_loc, 1, ws, (const __nv_bfloat16*)rows, p->H, p->ffn_path == 1 ? nullptr : p->Xp, p->cs, rowmap);
    p->launches += 3;
    // an expert receives at most one row per token of the step: m_e <= min(R, tokens_global)
    return expert_ffn(p, layer, ws, rows, R, 1, y_rows, ev, false,
                      (int)std::min<int64_t>(R, tokens_global > 0 ? tokens_global : R));
}

extern "C" dx_status dx_moe_forward_routed(dx_pool p, int32_t layer, const void* rows, int32_t R, const void* meta,
                                           void* y_rows, int64_t tokens_global) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    return routed_impl(p, layer, rows, R, meta, y_rows, tokens_global);
}

// Source side of the in-library EP layer: routing over the global experts and the placement (entries sorted by
// expert = grouped by owner), then the f-2 deduplication: one x row per (token, owner) into ep_send_rows, per-entry
// metadata {local expert, gate bits, row within the owner block} into ep_send_meta, and the per-owner triples
// {unique rows, entries, T} into ep_pairs[0 .. 3G).
static dx_status ep_dispatch_dedup(dx_pool p, int layer, const void* x, int T, const void* router_w,
                                   const float* router_bias, const float* logits, int32_t* topk_idx, float* topk_gate) {
    const int G = p->cfg.ep_size;
    p->ep_T = T;
    if (T == 0) {
        DX_CUDA(cudaMemsetAsync(p->ep_pairs, 0, sizeof(int32_t) * 3 * G, p->cs));
        return DX_OK;
    }
    RouteWs ws = p->ws_src;
    if (topk_idx) ws.idx = topk_idx;
    if (topk_gate) ws.gate = topk_gate;
    p->ws_src_live = ws;
    const float* lg = logits;
    if (router_w) {
        launch_router((const __nv_bfloat16*)x, (const __nv_bfloat16*)router_w, router_bias, T, p->E, p->H, ws.logits,
                      p->cs);
        lg = ws.logits;
        p->launches += 1;
    }
    const u64 nob[2][2] = {{0, 0}, {0, 0}};
    launch_route(lg, T, p->E, p->k, 0, ws, nullptr, nullptr, nullptr, nob, p->cs);
    launch_place(T, p->E, p->k, ws, nullptr, p->H, nullptr, p->cs);          // perm / inv only
    launch_dedup_dispatch(ws, T, p->k, p->E_loc, G, (const __nv_bfloat16*)x, p->H, p->ep_mark, p->ep_pairs,
                          p->ep_send_rows, p->ep_send_meta, p->cs);
    p->launches += 7;
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "EP dispatch launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

// Host bookkeeping of one local pool's exchange: rows (deduplicated) and entries to / from every peer.
struct EpPlan {
    std::vector<int> su, se, suoff, seoff, ru, re, ruoff, reoff;
    int64_t tokens_global = 0;
    int R = 0, U = 0;
};
static void ep_plan_from(int G, const int32_t* send3, const int32_t* recv3, EpPlan& q) {
    q.su.assign(G, 0); q.se.assign(G, 0); q.suoff.assign(G + 1, 0); q.seoff.assign(G + 1, 0);
    q.ru.assign(G, 0); q.re.assign(G, 0); q.ruoff.assign(G + 1, 0); q.reoff.assign(G + 1, 0);
    q.tokens_global = 0;
    for (int r = 0; r < G; ++r) {
        q.su[r] = send3[3 * r]; q.se[r] = send3[3 * r + 1];
        q.ru[r] = recv3[3 * r]; q.re[r] = recv3[3 * r + 1];
        q.tokens_global += recv3[3 * r + 2];
        q.suoff[r + 1] = q.suoff[r] + q.su[r]; q.seoff[r + 1] = q.seoff[r] + q.se[r];
        q.ruoff[r + 1] = q.ruoff[r] + q.ru[r]; q.reoff[r + 1] = q.reoff[r] + q.re[r];
    }
    q.R = q.reoff[G];
    q.U = q.ruoff[G];
}

// One expert-parallel layer (SURVEY §8(e) collective v1 + f-2 row deduplication) for n local pools: n = 1 with an
// NCCL communicator (one process per GPU), or all G ranks' pools of a local group (one process, one device, the
// exchange done by device copies).  Dispatch, the count exchange and ONE host synchronisation, the exchange of
// deduplicated rows and per-entry metadata, the owner-side FFN (hotness counted there with B_tot = the global
// token count), the return of one result row per entry, the rank-order combine (and fold).
static dx_status ep_layer(dx_pool* P, int n, int layer, const void* const* x, const int* T, const void* const* rw,
                          const float* const* rb, const float* const* lg, void* const* y, int32_t* const* topk_idx,
                          float* const* topk_gate, bool fuse_fold) {
    dx_pool p0 = P[0];
    const int G = p0->cfg.ep_size, k = p0->k, H = p0->H;
    const bool nccl = p0->comm != nullptr;
    DX_CHECK(nccl ? n == 1 : n == G, DX_ERR_INVALID_ARG, "an EP group call needs all %d ranks' pools (got %d)", G, n);
    for (int r = 0; r < n; ++r) {
        DX_CHECK(P[r] && (P[r]->comm || P[r]->ep_group) && P[r]->cfg.ep_size == G, DX_ERR_INVALID_ARG,
                 "pool %d is not an EP pool of size %d", r, G);
        DX_CHECK(nccl || (P[r]->cfg.ep_rank == r && P[r]->cs == p0->cs), DX_ERR_INVALID_ARG,
                 "local group: pool %d must have ep_rank %d and share the first pool's compute stream", r, r);
        DX_CHECK(layer >= 0 && layer < P[r]->L, DX_ERR_RANGE, "layer %d out of range", layer);
        DX_CHECK(T[r] >= 0 && T[r] <= P[r]->cfg.max_tokens, DX_ERR_RANGE, "T=%d outside [0, max_tokens]", T[r]);
        DX_CHECK(T[r] == 0 || (x[r] && y[r] && ((rw && rw[r]) != (lg && lg[r]))), DX_ERR_INVALID_ARG,
                 "pool %d: null x/y or not exactly one of router_w / logits", r);
        dx_status st = poll_transfers(P[r]);
        if (st != DX_OK) return st;
    }
    // 1. dispatch
    for (int r = 0; r < n; ++r) {
        dx_status st = ep_dispatch_dedup(P[r], layer, x[r], T[r], rw ? rw[r] : nullptr, rb ? rb[r] : nullptr,
                                         lg ? lg[r] : nullptr, topk_idx ? topk_idx[r] : nullptr,
                                         topk_gate ? topk_gate[r] : nullptr);
        if (st != DX_OK) return st;
    }
    // 2. counts: {unique rows, entries, T} per peer, then the host synchronisation
    std::vector<EpPlan> plan(n);
    if (nccl) {
        dx_pool p = p0;
        dx_status st = ep_nccl_exchange_counts(p->comm, G, 3, p->ep_pairs, p->ep_pairs + 3 * G, p->cs);
        if (st != DX_OK) return st;
        DX_CUDA(cudaMemcpyAsync(p->ep_pairs_host, p->ep_pairs, sizeof(int32_t) * 6 * G, cudaMemcpyDeviceToHost, p->cs));
        DX_CUDA(cudaStreamSynchronize(p->cs));
        ep_plan_from(G, p->ep_pairs_host, p->ep_pairs_host + 3 * G, plan[0]);
    } else {
        for (int r = 0; r < n; ++r)
            DX_CUDA(cudaMemcpyAsync(P[r]->ep_pairs_host, P[r]->ep_pairs, sizeof(int32_t) * 3 * G, cudaMemcpyDeviceToHost,
                                    p0->cs));
        DX_CUDA(cudaStreamSynchronize(p0->cs));
        for (int d = 0; d < n; ++d) {
            std::vector<int32_t> recv3(3 * G);
            for (int s = 0; s < n; ++s)
                for (int c = 0; c < 3; ++c) recv3[3 * s + c] = P[s]->ep_pairs_host[3 * d + c];
            ep_plan_from(G, P[d]->ep_pairs_host, recv3.data(), plan[d]);
        }
    }
    for (int r = 0; r < n; ++r) {
        DX_CHECK(plan[r].seoff[G] == T[r] * k, DX_ERR_INVALID_ARG, "internal: %d entries dispatched != T*k = %d",
                 plan[r].seoff[G], T[r] * k);
        DX_CHECK((size_t)plan[r].R <= P[r]->n_ent, DX_ERR_RANGE,
                 "received %d entries > workspace %zu (max_tokens must be the same on every rank)", plan[r].R, P[r]->n_ent);
        P[r]->ep_rows_sent += (u64)plan[r].suoff[G];
        P[r]->ep_entries_sent += (u64)plan[r].seoff[G];
    }
    // 3. rows + metadata
    if (nccl) {
        dx_pool p = p0;
        const EpPlan& q = plan[0];
        dx_status st = ep_nccl_exchange_rows(p->comm, G, H, p->ep_send_rows, q.su.data(), q.suoff.data(), p->ep_recv_rows,
                                             q.ru.data(), q.ruoff.data(), p->ep_send_meta, q.se.data(), q.seoff.data(),
                                             p->ep_recv_meta, q.re.data(), q.reoff.data(), 4, p->cs);
        if (st != DX_OK) return st;
    } else {
        for (int s = 0; s < n; ++s)
            for (int d = 0; d < n; ++d) {
                const EpPlan &qs = plan[s], &qd = plan[d];
                if (qs.su[d] > 0)
                    DX_CUDA(cudaMemcpyAsync(P[d]->ep_recv_rows + (size_t)qd.ruoff[s] * H,
                                            P[s]->ep_send_rows + (size_t)qs.suoff[d] * H, (size_t)qs.su[d] * H * 2,
                                            cudaMemcpyDeviceToDevice, p0->cs));
                if (qs.se[d] > 0)
                    DX_CUDA(cudaMemcpyAsync(P[d]->ep_recv_meta + qd.reoff[s], P[s]->ep_send_meta + qs.seoff[d],
                                            (size_t)qs.se[d] * sizeof(int4), cudaMemcpyDeviceToDevice, p0->cs));
            }
    }
    // 4. owner-side FFN on the received entries (rows gathered through the dedup row map)
    for (int r = 0; r < n; ++r) {
        dx_pool p = P[r];
        const EpPlan& q = plan[r];
        launch_dedup_fix(p->ep_recv_meta, q.R, G, q.reoff.data(), q.ruoff.data(), p->ep_meta2, p->ep_rowmap, p->cs);
        p->launches += 1;
        dx_status st = routed_impl(p, layer, p->ep_recv_rows, q.R, p->ep_meta2, p->ep_y_rows, q.tokens_global,
                                   p->ep_rowmap);
        if (st != DX_OK) return st;
    }
    // 5. one result row per entry back to its source, in the source's dispatch order
    if (nccl) {
        dx_pool p = p0;
        const EpPlan& q = plan[0];
        dx_status st = ep_nccl_exchange_rows(p->comm, G, H, p->ep_y_rows, q.re.data(), q.reoff.data(), p->ep_back_rows,
                                             q.se.data(), q.seoff.data(), nullptr, nullptr, nullptr, nullptr, nullptr,
                                             nullptr, 0, p->cs);
        if (st != DX_OK) return st;
    } else {
        for (int s = 0; s < n; ++s)
            for (int d = 0; d < n; ++d) {
                const EpPlan &qs = plan[s], &qd = plan[d];
                if (qs.se[d] > 0)
                    DX_CUDA(cudaMemcpyAsync(P[s]->ep_back_rows + (size_t)qs.seoff[d] * H,
                                            P[d]->ep_y_rows + (size_t)qd.reoff[s] * H, (size_t)qs.se[d] * H * 2,
                                            cudaMemcpyDeviceToDevice, p0->cs));
            }
    }
    // 6. combine (+ fold)
    for (int r = 0; r < n; ++r) {
        dx_pool p = P[r];
        if (fuse_fold) {
            FoldReq req;
            dx_status st = fold_prepare(p, layer, &req);
            if (st != DX_OK) return st;
            launch_combine(p->ep_back_rows, T[r], k, H, (__nv_bfloat16*)y[r], p->cs, p->ws_src_live.inv, &p->ctrl, &req);
        } else if (T[r] > 0) {
            launch_combine(p->ep_back_rows, T[r], k, H, (__nv_bfloat16*)y[r], p->cs, p->ws_src_live.inv);
        }
        p->launches += 1;
    }
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "EP layer launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

static dx_status ep_forward(dx_pool p, int layer, const void* x, int T, const void* router_w, const float* router_bias,
                            const float* logits, void* y, int32_t* topk_idx, float* topk_gate, bool fuse_fold) {
    DX_CHECK(p->comm, DX_ERR_INVALID_ARG, "a local-group EP pool runs through dx_moe_step_group");
    return ep_layer(&p, 1, layer, &x, &T, router_w ? &router_w : nullptr, router_w ? &router_bias : nullptr,
                    logits ? &logits : nullptr, &y, topk_idx ? &topk_idx : nullptr, topk_gate ? &topk_gate : nullptr,
                    fuse_fold);
}

extern "C" dx_status dx_moe_step_group(dx_pool* pools, int32_t n, int32_t layer, const void* const* x, const int32_t* T,
                                       const void* const* router_w, const float* const* router_bias,
                                       const float* const* logits, void* const* y) {
    DX_CHECK(pools && n >= 1 && n <= 8 && x && T && y, DX_ERR_INVALID_ARG, "bad group arguments");
    dx_status st = ep_layer(pools, n, layer, x, T, router_w, router_bias, logits, y, nullptr, nullptr, true);
    if (st != DX_OK) return st;
    for (int r = 0; r < n; ++r) {
        st = dx_plan_precision(pools[r], layer, nullptr);
        if (st != DX_OK) return st;
    }
    return DX_OK;
}

extern "C" dx_status dx_ep_traffic(dx_pool p, uint64_t* rows_sent, uint64_t* entries_sent) {
    DX_CHECK(p && rows_sent && entries_sent, DX_ERR_INVALID_ARG, "null argument");
    *rows_sent = p->ep_rows_sent;
    *entries_sent = p->ep_entries_sent;
    return DX_OK;
}

extern "C" dx_status dx_ep_combine(dx_pool p, int32_t layer, const void* back_rows, int32_t T, void* y) {
    CHECK_LAYER(p, layer);
    DX_CHECK(p->cfg.ep_size > 1 || p->comm, DX_ERR_INVALID_ARG, "dx_ep_combine needs ep_size > 1");
    DX_CHECK(T == p->ep_T, DX_ERR_INVALID_ARG, "T=%d does not match the last dispatch (%d)", T, p->ep_T);
    if (T == 0) return DX_OK;
    DX_CHECK(back_rows && y, DX_ERR_INVALID_ARG, "null buffer");
    launch_combine((const __nv_bfloat16*)back_rows, T, p->k, p->H, (__nv_bfloat16*)y, p->cs, p->ws_src_live.inv);
    p->launches += 1;
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "combine launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

// Host side of a10/a14: the step count, B_tot and -- when transitions publish at the new step -- the
// compute stream's wait for the side stream (the exposed switch time, if any, is spent in that wait).
static dx_status fold_prepare(dx_pool p, int layer, FoldReq* req) {
    const u64 B = p->pend_tokens[layer];
    p->pend_tokens[layer] = 0;
    const i64 t_new = p->t[layer] + 1;
    if (p->publish_at[layer] == t_new) {
        dx_status st = poll_transfers(p, layer);        // the plan's transfers must have been issued by now
        if (st != DX_OK) return st;
        st = io_wait(p, layer);                          // (SSD tier: the I/O thread's hand-over too)
        if (st != DX_OK) return st;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (p->profiling) {
            e0 = prof_event(p);
            e1 = prof_event(p);
            p->prof_wait_ev.push_back(e0);
            p->prof_wait_ev.push_back(e1);
            DX_CUDA(cudaEventRecord(e0, p->cs));
        }
        // a side stream that already finished needs no cross-stream dependency (which would break the PDL chain)
        const cudaError_t q = cudaEventQuery(p->ev_side[layer]);
        if (q == cudaErrorNotReady) DX_CUDA(cudaStreamWaitEvent(p->cs, p->ev_side[layer], 0));
        else DX_CHECK(q == cudaSuccess, DX_ERR_CUDA, "side-stream event: %s", cudaGetErrorString(q));
        if (e1) DX_CUDA(cudaEventRecord(e1, p->cs));
        p->publish_at[layer] = -1;
    }
    p->t[layer] = t_new;
    req->layer = layer;
    req->B_tot = B;
    return DX_OK;
}

static dx_status fold(dx_pool p, int layer) {
    FoldReq req;
    dx_status st = fold_prepare(p, layer, &req);
    if (st != DX_OK) return st;
    launch_fold(p->ctrl, layer, req.B_tot, p->cs);
    p->launches += 1;
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "fold launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

extern "C" dx_status dx_hotness_update(dx_pool p, int32_t layer) {
    CHECK_LAYER(p, layer);
    return fold(p, layer);
}

extern "C" dx_status dx_hotness_update_from(dx_pool p, int32_t layer, const int32_t* idx, const float* gate,
                                            int32_t T) {
    CHECK_LAYER(p, layer);
    DX_CHECK(T >= 0 && (T == 0 || (idx && gate)), DX_ERR_INVALID_ARG, "bad idx/gate");
    const size_t base = (size_t)layer * p->E_loc;
    if (T > 0) {
        DX_CUDA(cudaMemsetAsync(p->err_flag, 0, 4, p->cs));
        launch_counts_from(idx, gate, T, p->E, p->E_loc, p->k, p->e_lo, p->ctrl.cnt + base, p->ctrl.mass + base,
                           p->err_flag, p->cs);
        p->launches += 1;
        int32_t err = 0;
        DX_CUDA(cudaMemcpyAsync(&err, p->err_flag, 4, cudaMemcpyDeviceToHost, p->cs));
        DX_CUDA(cudaStreamSynchronize(p->cs));
        DX_CHECK(err == 0, err == 1 ? DX_ERR_INVALID_ARG : DX_ERR_RANGE,
                 err == 1 ? "duplicate expert within one token (SPEC.md:144)" : "expert id out of range");
    }
    p->pend_tokens[layer] += (u64)T;
    return fold(p, layer);
}

static XferArgs xfer_args(dx_pool p, int layer) {
    XferArgs x;
    x.layer_base = p->weights + (size_t)layer * p->layer_bytes;
    x.hi_base = p->hi_base;
    x.hi = p->hi;
    x.lo = p->lo;
    x.hi_img = p->hi_img_dev + (size_t)layer * p->E_loc;
    x.H = p->H; x.I = p->I; x.g = p->g;
    return x;
}

static dx_status read_plan(dx_pool p, int layer, dx_plan* out) {
    DX_CUDA(cudaStreamSynchronize(p->cs));
    int32_t n = 0;
    DX_CUDA(cudaMemcpy(&n, p->ctrl.plan_n + layer, 4, cudaMemcpyDeviceToHost));
    std::vector<int4> cmds(n > 0 ? n : 1);
    if (n > 0) DX_CUDA(cudaMemcpy(cmds.data(), p->ctrl.plan_cmd + (size_t)layer * p->E_loc, n * sizeof(int4), cudaMemcpyDeviceToHost));
    out->n = n < DX_MAX_CMDS ? n : DX_MAX_CMDS;
    for (int i = 0; i < out->n; ++i) {
        out->cmd[i].expert = cmds[i].x;
        out->cmd[i].dir = cmds[i].y;
        out->cmd[i].dst_slot = cmds[i].z;
        out->cmd[i].src_slot = cmds[i].w;
    }
    return DX_OK;
}

// a12/a13 of one layer's runtime plan on the side stream: the demotion kernel (on-device quantisation) and one
// copy-engine H2D per promotion from the pinned HIGH image into its destination block; ev_side marks them done.
static dx_status issue_transfers(dx_pool p, int layer) {
    const size_t E = (size_t)p->E_loc;
    if (p->pf_pending[layer]) {                    // the layer's prefetch copies go first on the side stream
        DX_CUDA(cudaEventSynchronize(p->ev_pf[layer]));
        dx_status st = issue_prefetch(p, layer);
        if (st != DX_OK) return st;
    }
    cudaEvent_t x0 = nullptr;
    if (p->profiling) {
        x0 = prof_event(p);
        p->prof_xfer_ev.push_back(x0);
        DX_CUDA(cudaEventRecord(x0, p->ss));
    }
    const int n = p->plan_n_host[layer];
    int nd = 0;
    for (int i = 0; i < n; ++i) nd += p->plan_host[layer * E + i].y == -1;
    // TIMING ATTRIBUTION ONLY (results wrong): DX_XFER_SKIP=1 skips the demotions' quantisation, =2 the promotions' copies
    static const int xfer_skip = [] { const char* e = getenv("DX_XFER_SKIP"); return e ? atoi(e) : 0; }();
    if (nd > 0 && xfer_skip != 1) {  // demotions: device quantisation on the second side stream, beside the copies
        DX_CUDA(cudaStreamWaitEvent(p->ss2, p->ev_planh[layer], 0));
        launch_transitions(p->ctrl, layer, xfer_args(p, layer), n, 3, p->ss2);
        DX_CUDA(cudaEventRecord(p->ev_dem, p->ss2));
        p->launches += 1;
    }
    const size_t bytes = p->hi.bits == 16 ? (size_t)3 * p->I * p->H * 2 : (size_t)p->hi.bytes;
    uint8_t* hi_region = p->weights + (size_t)layer * p->layer_bytes + p->hi_base;
    u64 np = 0;
    if (p->io_thread.joinable()) {
        // hand the promotions' copies (f-4: and the SSD reads) to the transfer thread; it records ev_side when they
        // are issued, so the host thread issuing the forwards never spends its time on them
        dx_pool_s::IoJob job{layer, {}, nd > 0, nullptr, nullptr};
        for (int i = 0; i < n; ++i) {
            const int4 cmd = p->plan_host[layer * E + i];
            if (cmd.y != 1) continue;
            bool hit = false;
            for (const int2& sg : p->staged[layer]) hit |= sg.x == cmd.x && sg.y == cmd.z;
            if (hit) { ++p->pf_hits; continue; }
            job.copies.emplace_back(layer * E + cmd.x, hi_region + (size_t)cmd.z * p->hi.bytes);
        }
        if (x0) {
            job.x1 = prof_event(p);
            p->prof_xfer_ev.push_back(job.x1);
            if (!job.copies.empty()) {
                job.xc = prof_event(p);
                p->prof_copy_ev.push_back(x0);
                p->prof_copy_ev.push_back(job.xc);
                p->prof_copy_bytes.push_back(job.copies.size() * bytes);
            }
        }
        {
            std::lock_guard<std::mutex> lk(p->io_mu);
            p->io_pending[layer] = 1;
            ++p->io_inflight;
            p->io_q.push_back(std::move(job));
        }
        p->io_cv.notify_all();
        p->staged[layer].clear();
        p->xfer_pending[layer] = 0;
        p->n_pending -= 1;
        return DX_OK;
    }
    for (int i = 0; i < n; ++i) {
        const int4 cmd = p->plan_host[layer * E + i];
        if (cmd.y != 1) continue;
        bool hit = false;                          // staged by the prefetch into this very block already
        for (const int2& sg : p->staged[layer]) hit |= sg.x == cmd.x && sg.y == cmd.z;
        if (hit) { ++p->pf_hits; continue; }
        if (xfer_skip == 2) continue;
        dx_status rc = copy_high_image(p, layer * E + cmd.x, hi_region + (size_t)cmd.z * p->hi.bytes, p->ss);
        if (rc != DX_OK) return rc;
        ++np;
    }
    if (x0 && np > 0) {
        cudaEvent_t xc = prof_event(p);
        DX_CUDA(cudaEventRecord(xc, p->ss));
        p->prof_copy_ev.push_back(x0);
        p->prof_copy_ev.push_back(xc);
        p->prof_copy_bytes.push_back(np * bytes);
    }
    if (nd > 0 && xfer_skip != 1) DX_CUDA(cudaStreamWaitEvent(p->ss, p->ev_dem, 0));
    if (x0) {
        cudaEvent_t x1 = prof_event(p);
        p->prof_xfer_ev.push_back(x1);
        DX_CUDA(cudaEventRecord(x1, p->ss));
    }
    DX_CUDA(cudaEventRecord(p->ev_side[layer], p->ss));
    p->staged[layer].clear();
    p->xfer_pending[layer] = 0;
    p->n_pending -= 1;
    return DX_OK;
}

// issue every pending layer's transfers whose plan has reached the host (non-blocking), or -- wait_layer >= 0 --
// that layer's unconditionally (it publishes now)
static dx_status poll_transfers(dx_pool p, int wait_layer) {
    if (p->n_pending == 0) return DX_OK;
    if (wait_layer >= 0 && p->xfer_pending[wait_layer]) {
        DX_CUDA(cudaEventSynchronize(p->ev_planh[wait_layer]));
        dx_status st = issue_transfers(p, wait_layer);
        if (st != DX_OK) return st;
    }
    for (int l = 0; l < p->L && p->n_pending > 0; ++l) {
        if (p->pf_pending[l]) {
            const cudaError_t q = cudaEventQuery(p->ev_pf[l]);
            if (q == cudaSuccess) {
                dx_status st = issue_prefetch(p, l);
                if (st != DX_OK) return st;
            } else if (q != cudaErrorNotReady) {
                dx_set_error("prefetch event: %s", cudaGetErrorString(q));
                return DX_ERR_CUDA;
            }
        }
        if (!p->xfer_pending[l]) continue;
        const cudaError_t q = cudaEventQuery(p->ev_planh[l]);
        if (q == cudaErrorNotReady) continue;
        DX_CHECK(q == cudaSuccess, DX_ERR_CUDA, "plan event: %s", cudaGetErrorString(q));
        dx_status st = issue_transfers(p, l);
        if (st != DX_OK) return st;
    }
    return DX_OK;
}

extern "C" dx_status dx_plan_precision(dx_pool p, int32_t layer, dx_plan* out) {
    CHECK_LAYER(p, layer);
    const i64 t = p->t[layer];
    const dx_config& c = p->cfg;
    if (out) { out->due = 0; out->finalize = 0; out->n = 0; out->step = t; out->publish_step = t; }
    if (!p->finalized[layer] && t == c.warmup_steps) {
        // §3.5: tau_h and the initial HIGH set, installed synchronously before serving continues
        launch_plan(p->ctrl, layer, 1, p->cs);
        launch_transitions(p->ctrl, layer, xfer_args(p, layer), p->E_loc, 1, p->cs);
        if (p->ssd_fd < 0) {
            launch_transitions(p->ctrl, layer, xfer_args(p, layer), p->E_loc, 2, p->cs);
        } else {
            // f-4: the initial HIGH set comes from the SSD tier through the DRAM cache (copy engine, in order
            // after the relayout moves on the compute stream)
            const size_t E = (size_t)p->E_loc;
            DX_CUDA(cudaMemcpyAsync(p->plan_n_host + layer, p->ctrl.plan_n + layer, 4, cudaMemcpyDeviceToHost, p->cs));
            DX_CUDA(cudaMemcpyAsync(p->plan_host + layer * E, p->ctrl.plan_cmd + layer * E, E * sizeof(int4),
                                    cudaMemcpyDeviceToHost, p->cs));
            DX_CUDA(cudaStreamSynchronize(p->cs));
            uint8_t* hi_region = p->weights + (size_t)layer * p->layer_bytes + p->hi_base;
            for (int i = 0; i < p->plan_n_host[layer]; ++i) {
                const int4 cmd = p->plan_host[layer * E + i];
                if (cmd.y != 1) continue;
                dx_status rc = copy_high_image(p, layer * E + cmd.x, hi_region + (size_t)cmd.z * p->hi.bytes, p->cs);
                if (rc != DX_OK) return rc;
            }
        }
        p->launches += 3;
        p->finalized[layer] = 1;
        if (out) {
            out->due = 1; out->finalize = 1;
            dx_status st = read_plan(p, layer, out);
            if (st != DX_OK) return st;
        }
        cudaError_t ce = cudaGetLastError();
        DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "finalize launch failed: %s", cudaGetErrorString(ce));
        return DX_OK;
    }
    if (!p->finalized[layer] || t <= c.warmup_steps || t % c.period != 0 || p->publish_at[layer] >= 0) return DX_OK;
    launch_plan(p->ctrl, layer, 0, p->cs);
    p->launches += 1;
    if (p->teleport) {
        DX_CUDA(cudaEventRecord(p->ev_side[layer], p->cs));
    } else {
        // the plan to pinned host memory, copied on the side stream (copies on the compute stream would break the
        // programmatic-dependent-launch chain of the forwards); the transfers are issued once the host sees it
        const size_t E = (size_t)p->E_loc;
        DX_CUDA(cudaEventRecord(p->ev_plandone[layer], p->cs));
        DX_CUDA(cudaStreamWaitEvent(p->ss, p->ev_plandone[layer], 0));
        DX_CUDA(cudaMemcpyAsync(p->plan_n_host + layer, p->ctrl.plan_n + layer, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                p->ss));
        DX_CUDA(cudaMemcpyAsync(p->plan_host + layer * E, p->ctrl.plan_cmd + layer * E, E * sizeof(int4),
                                cudaMemcpyDeviceToHost, p->ss));
        DX_CUDA(cudaEventRecord(p->ev_planh[layer], p->ss));
        p->xfer_pending[layer] = 1;
        p->n_pending += 1;
    }
    p->publish_at[layer] = t + c.publish_lag;
    if (out) {
        out->due = 1;
        out->publish_step = t + c.publish_lag;
        dx_status st = read_plan(p, layer, out);
        if (st != DX_OK) return st;
    }
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "plan launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

static dx_status manual(dx_pool p, int layer, const int32_t* experts, int n, int dir) {
    CHECK_LAYER(p, layer);
    DX_CHECK(n >= 0 && n <= 1024 && (n == 0 || experts), DX_ERR_INVALID_ARG, "bad expert list");
    if (n == 0) return DX_OK;
    DX_CHECK(p->finalized[layer], DX_ERR_NOT_READY, "warm-up of layer %d not finished", layer);
    const i64 due = p->t[layer] + p->cfg.publish_lag;
    DX_CHECK(p->publish_at[layer] < 0 || p->publish_at[layer] == due, DX_ERR_BUSY,
             "layer %d has transitions publishing at a different step", layer);
    {
        dx_status st = poll_transfers(p, layer);     // a pending plan's demotions read plan_cmd: issue them first
        if (st != DX_OK) return st;
    }
    std::vector<int2> cmds(n);
    for (int i = 0; i < n; ++i) cmds[i] = make_int2(experts[i], dir);
    // k_manual rewrites the layer's command list (plan_cmd / plan_n): transitions issued earlier for this
    // layer must have finished reading it on the side stream first
    if (p->publish_at[layer] >= 0) {
        dx_status st = io_wait(p, layer);
        if (st != DX_OK) return st;
        DX_CUDA(cudaStreamWaitEvent(p->cs, p->ev_side[layer], 0));
    }
    DX_CUDA(cudaMemcpyAsync(p->manual_cmds, cmds.data(), n * sizeof(int2), cudaMemcpyHostToDevice, p->cs));
    launch_manual(p->ctrl, layer, p->manual_cmds, n, p->manual_status, p->cs);
    DX_CUDA(cudaEventRecord(p->ev_plan, p->cs));
    DX_CUDA(cudaStreamWaitEvent(p->ss, p->ev_plan, 0));
    if (p->ssd_fd < 0) {
        launch_transitions(p->ctrl, layer, xfer_args(p, layer), n, 0, p->ss);
    } else {                                          // f-4: promotions through the SSD tier's DRAM cache
        const size_t E = (size_t)p->E_loc;
        launch_transitions(p->ctrl, layer, xfer_args(p, layer), n, 3, p->ss);     // demotions
        DX_CUDA(cudaMemcpyAsync(p->plan_n_host + layer, p->ctrl.plan_n + layer, 4, cudaMemcpyDeviceToHost, p->cs));
        DX_CUDA(cudaMemcpyAsync(p->plan_host + layer * E, p->ctrl.plan_cmd + layer * E, E * sizeof(int4),
                                cudaMemcpyDeviceToHost, p->cs));
        DX_CUDA(cudaStreamSynchronize(p->cs));
        uint8_t* hi_region = p->weights + (size_t)layer * p->layer_bytes + p->hi_base;
        for (int i = 0; i < p->plan_n_host[layer]; ++i) {
            const int4 cmd = p->plan_host[layer * E + i];
            if (cmd.y != 1) continue;
            dx_status rc = copy_high_image(p, layer * E + cmd.x, hi_region + (size_t)cmd.z * p->hi.bytes, p->ss);
            if (rc != DX_OK) return rc;
        }
    }
    DX_CUDA(cudaEventRecord(p->ev_side[layer], p->ss));
    p->launches += 2;
    p->publish_at[layer] = due;
    std::vector<int32_t> stv(n);
    DX_CUDA(cudaMemcpyAsync(stv.data(), p->manual_status, n * 4, cudaMemcpyDeviceToHost, p->cs));
    DX_CUDA(cudaStreamSynchronize(p->cs));
    for (int i = 0; i < n; ++i) {
        switch (stv[i]) {
            case 0: break;
            case 1: dx_set_error("expert %d already at that tier", experts[i]); return DX_ERR_INVALID_ARG;
            case 2: dx_set_error("expert %d out of range", experts[i]); return DX_ERR_RANGE;
            case 4: dx_set_error("no free block for expert %d (deferred)", experts[i]); return DX_ERR_POOL_EXHAUSTED;
            case 5: dx_set_error("expert %d has a transition in flight", experts[i]); return DX_ERR_BUSY;
            default: return DX_ERR_LEDGER;
        }
    }
    return DX_OK;
}

extern "C" dx_status dx_promote(dx_pool p, int32_t layer, const int32_t* experts, int32_t n) {
    return manual(p, layer, experts, n, 1);
}
extern "C" dx_status dx_demote(dx_pool p, int32_t layer, const int32_t* experts, int32_t n) {
    return manual(p, layer, experts, n, -1);
}

extern "C" dx_status dx_sync(dx_pool p) {
    DX_CHECK(p, DX_ERR_INVALID_ARG, "null pool");
    for (int l = 0; l < p->L; ++l) {
        if (p->pf_pending[l]) {
            DX_CUDA(cudaEventSynchronize(p->ev_pf[l]));
            dx_status st = issue_prefetch(p, l);
            if (st != DX_OK) return st;
        }
        if (!p->xfer_pending[l]) continue;
        dx_status st = poll_transfers(p, l);
        if (st != DX_OK) return st;
    }
    {
        dx_status st = io_wait(p, -1);
        if (st != DX_OK) return st;
    }
    DX_CUDA(cudaStreamSynchronize(p->ss2));
    DX_CUDA(cudaStreamSynchronize(p->ss));
    DX_CUDA(cudaStreamSynchronize(p->cs));
    DX_CUDA(cudaGetLastError());
    int32_t err = 0;
    DX_CUDA(cudaMemcpy(&err, p->dev_err, 4, cudaMemcpyDeviceToHost));
    if (err) {
        DX_CUDA(cudaMemset(p->dev_err, 0, 4));
        dx_set_error("dx_moe_forward_routed received an expert id outside [0, E_loc) (row output set to 0)");
        return DX_ERR_RANGE;
    }
    return DX_OK;
}

extern "C" dx_status dx_get_table(dx_pool p, int32_t layer, int32_t* tier, int32_t* slot, uint32_t* version,
                                  int32_t* in_flight) {
    CHECK_LAYER(p, layer);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    const size_t b = (size_t)layer * p->E_loc, n = p->E_loc;
    if (tier) DX_CUDA(cudaMemcpy(tier, p->ctrl.tier + b, n * 4, cudaMemcpyDeviceToHost));
    if (slot) DX_CUDA(cudaMemcpy(slot, p->ctrl.slot + b, n * 4, cudaMemcpyDeviceToHost));
    if (version) DX_CUDA(cudaMemcpy(version, p->ctrl.version + b, n * 4, cudaMemcpyDeviceToHost));
    if (in_flight) DX_CUDA(cudaMemcpy(in_flight, p->ctrl.pend_dir + b, n * 4, cudaMemcpyDeviceToHost));
    return DX_OK;
}

extern "C" dx_status dx_query_expert(dx_pool p, int32_t layer, int32_t e, int32_t* tier, int32_t* slot,
                                     uint32_t* version, int32_t* in_flight) {
    CHECK_LAYER(p, layer);
    DX_CHECK(e >= 0 && e < p->E_loc, DX_ERR_RANGE, "expert %d out of range", e);
    std::vector<int32_t> tr(p->E_loc), sl(p->E_loc), fl(p->E_loc);
    std::vector<uint32_t> vr(p->E_loc);
    dx_status st = dx_get_table(p, layer, tr.data(), sl.data(), vr.data(), fl.data());
    if (st != DX_OK) return st;
    if (tier) *tier = tr[e];
    if (slot) *slot = sl[e];
    if (version) *version = vr[e];
    if (in_flight) *in_flight = fl[e];
    return DX_OK;
}

extern "C" dx_status dx_occupancy(dx_pool p, int32_t layer, int32_t* used_hi, int32_t* cap_hi, int32_t* used_lo,
                                  int32_t* cap_lo) {
    CHECK_LAYER(p, layer);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    const int n = p->E_loc + p->cfg.n_spare;
    std::vector<int32_t> lo(n), hi(n);
    int32_t clo, chi;
    DX_CUDA(cudaMemcpy(lo.data(), p->ctrl.lo_owner + (size_t)layer * n, n * 4, cudaMemcpyDeviceToHost));
    DX_CUDA(cudaMemcpy(hi.data(), p->ctrl.hi_owner + (size_t)layer * n, n * 4, cudaMemcpyDeviceToHost));
    DX_CUDA(cudaMemcpy(&clo, p->ctrl.cap_lo + layer, 4, cudaMemcpyDeviceToHost));
    DX_CUDA(cudaMemcpy(&chi, p->ctrl.cap_hi + layer, 4, cudaMemcpyDeviceToHost));
    int uh = 0, ul = 0;
    for (int i = 0; i < chi; ++i) uh += hi[i] >= 0;
    for (int i = 0; i < clo; ++i) ul += lo[i] >= 0;
    if (used_hi) *used_hi = uh;
    if (cap_hi) *cap_hi = chi;
    if (used_lo) *used_lo = ul;
    if (cap_lo) *cap_lo = clo;
    return DX_OK;
}

extern "C" dx_status dx_get_hotness(dx_pool p, int32_t layer, double* S, uint32_t* cnt, uint64_t* mass,
                                    double* tau_h, int32_t* n_hot, int64_t* step) {
    CHECK_LAYER(p, layer);
    DX_CUDA(cudaStreamSynchronize(p->cs));
    const size_t b = (size_t)layer * p->E_loc, n = p->E_loc;
    if (S) DX_CUDA(cudaMemcpy(S, p->ctrl.S + b, n * 8, cudaMemcpyDeviceToHost));
    if (cnt) DX_CUDA(cudaMemcpy(cnt, p->ctrl.cnt + b, n * 4, cudaMemcpyDeviceToHost));
    if (mass) DX_CUDA(cudaMemcpy(mass, p->ctrl.mass + b, n * 8, cudaMemcpyDeviceToHost));
    if (tau_h) DX_CUDA(cudaMemcpy(tau_h, p->ctrl.tau + layer, 8, cudaMemcpyDeviceToHost));
    if (n_hot) *n_hot = p->info.n_hot;
    if (step) *step = p->t[layer];
    return DX_OK;
}

extern "C" dx_status dx_export_expert(dx_pool p, int32_t layer, int32_t e, void* host_out, int64_t cap,
                                      int64_t* written) {
    CHECK_LAYER(p, layer);
    DX_CHECK(e >= 0 && e < p->E_loc, DX_ERR_RANGE, "expert %d out of range", e);
    DX_CHECK(host_out, DX_ERR_INVALID_ARG, "null output");
    int32_t tier, slot;
    dx_status st = dx_query_expert(p, layer, e, &tier, &slot, nullptr, nullptr);
    if (st != DX_OK) return st;
    const SlotLayout& Ls = tier ? p->hi : p->lo;
    const uint8_t* src = p->weights + (size_t)layer * p->layer_bytes + (tier ? p->hi_base + (i64)slot * p->hi.bytes
                                                                             : (i64)slot * p->lo.bytes);
    const i64 n = (i64)p->I * p->H, n3 = 3 * n;
    const i64 need = Ls.bits == 16 ? n3 * 2 : n3 + n3 / p->g * 3;
    DX_CHECK(cap >= need, DX_ERR_INVALID_ARG, "output buffer too small (%lld < %lld)", (long long)cap, (long long)need);
    std::vector<uint8_t> img(Ls.bytes);
    DX_CUDA(cudaMemcpy(img.data(), src, Ls.bytes, cudaMemcpyDeviceToHost));
    uint8_t* o = (uint8_t*)host_out;
    if (Ls.bits == 16) {
        memcpy(o, img.data(), n3 * 2);
    } else {
        // slots hold the pair-interleaved packing (dx_quant.cuh): un-interleave to canonical u8 codes
        const int W = 32 / Ls.bits, mask = (1 << Ls.bits) - 1;
        for (int m = 0; m < 3; ++m) {
            const uint8_t* codes = img.data() + m * Ls.codes_stride;
            for (i64 i = 0; i < n; ++i) {
                uint32_t word;
                memcpy(&word, codes + (i / W) * 4, 4);
                const int e = (int)(i % W), slot = (e & 1) ? W / 2 + e / 2 : e / 2;
                o[m * n + i] = (word >> (Ls.bits * slot)) & mask;
            }
            memcpy(o + n3 + m * (n / p->g) * 2, img.data() + Ls.scales_off + m * Ls.scales_stride, (n / p->g) * 2);
            memcpy(o + n3 + n3 / p->g * 2 + m * (n / p->g), img.data() + Ls.zeros_off + m * Ls.zeros_stride, n / p->g);
        }
    }
    if (written) *written = need;
    return DX_OK;
}

extern "C" dx_status dx_quantize(const void* w, int64_t N, int64_t K, int32_t g, int32_t bits, void* codes,
                                 void* scales, void* zeros, void* stream) {
    DX_CHECK(w && codes && scales && zeros, DX_ERR_INVALID_ARG, "null pointer");
    DX_CHECK((g == 32 || g == 64 || g == 128) && K % g == 0 && N >= 0 && (bits == 4 || bits == 2),
             DX_ERR_INVALID_ARG, "bad shape/bits");
    launch_quantize(w, 16, nullptr, nullptr, N, K, g, bits, (uint8_t*)codes, (__nv_bfloat16*)scales,
                    (uint8_t*)zeros, (cudaStream_t)stream);
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "quantize launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}

extern "C" dx_status dx_dequantize(const void* codes, const void* scales, const void* zeros, int64_t N, int64_t K,
                                   int32_t g, int32_t bits, void* w, void* stream) {
    DX_CHECK(w && codes && scales && zeros, DX_ERR_INVALID_ARG, "null pointer");
    DX_CHECK((g == 32 || g == 64 || g == 128) && K % g == 0 && K % 8 == 0 && N >= 0 && (bits == 4 || bits == 2),
             DX_ERR_INVALID_ARG, "bad shape/bits");
    launch_dequantize((const uint8_t*)codes, (const __nv_bfloat16*)scales, (const uint8_t*)zeros, N, K, g, bits,
                      (__nv_bfloat16*)w, (cudaStream_t)stream);
    cudaError_t ce = cudaGetLastError();
    DX_CHECK(ce == cudaSuccess, DX_ERR_CUDA, "dequantize launch failed: %s", cudaGetErrorString(ce));
    return DX_OK;
}
