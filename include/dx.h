/*
 * dx.h -- C ABI of the DynaExq hot path on B200 (sm_100a).
 *
 * DynaExq (arXiv 2511.15015, /root/reference/PAPER.md): a hybrid-precision MoE expert layer whose
 * experts live in a fragmentation-free slot pool at a HIGH or LOW precision tier chosen at run
 * time by an EMA-hotness controller under an HBM budget.  Citations: PAPER.md:line; readings of
 * ambiguous passages are DESIGN.md §2 (R-*).
 *
 * Conventions for every entry point
 *  - Plain C types only; no torch types.  Device pointers are CUDA device (or UVA-mapped) memory
 *    ordered on the pool's compute stream; host pointers are ordinary host memory.
 *  - Every call returns a dx_status; nothing is thrown across the ABI.  On failure
 *    dx_last_error() returns a thread-local message (valid until the next failing call).
 *  - One host thread mutates a pool at a time (SPEC.md:197 single mutator); pools are independent.
 *  - The library owns the device arena: exactly ONE cudaMalloc per pool, in dx_pool_create, and no
 *    device allocation afterwards ("avoids runtime cudaMalloc calls").
 */
#ifndef DYNAEXQ_DX_H
#define DYNAEXQ_DX_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DX_OK = 0,
    DX_ERR_INVALID_ARG = 1,        /* malformed argument / wrong tier for a command */
    DX_ERR_RANGE = 2,              /* layer / expert / n_hot out of range */
    DX_ERR_INFEASIBLE_BUDGET = 3,  /* budget < (N+s)*S_l + s*S_h per layer */
    DX_ERR_POOL_EXHAUSTED = 4,     /* no free block; the command is deferred, pool never grows */
    DX_ERR_BUSY = 5,               /* expert already has a transition in flight */
    DX_ERR_LEDGER = 6,             /* ledger corruption (double free / foreign block), fatal */
    DX_ERR_NOT_READY = 7,          /* operation needs the warm-up to have finished */
    DX_ERR_CUDA = 8,
    DX_ERR_NCCL = 9,
    DX_ERR_OOM = 10
} dx_status;

/* Precision of a tier: 16 = bf16, 4 = int4, 2 = int2 (group-wise asymmetric, DESIGN.md R-Q1).
 * Pairs used by the paper: (16,4) for Qwen3-30B-A3B, (4,2) for Qwen3-Next-80B-A3B. */
typedef struct {
    int32_t num_layers;         /* L */
    int32_t num_experts;        /* global E (= N, the paper's m) */
    int32_t top_k;              /* k */
    int32_t hidden;             /* H (multiple of group_size and of 256) */
    int32_t inter;              /* I, expert intermediate size (multiple of group_size and of 64) */
    int32_t group_size;         /* g: 128, or 32 for tiny shapes */
    int32_t high_bits;          /* 16 or 4 */
    int32_t low_bits;           /* 4 or 2, < high_bits */
    uint64_t expert_budget_bytes; /* per GPU, all layers; M = floor(budget / L) per layer */
    int32_t n_spare;            /* spare blocks per tier per layer: the transient buffer */
    double  ema_alpha;          /* alpha of Eq. 2 */
    int32_t period;             /* Tp: plan when t ≡ 0 mod Tp (Alg. 1) */
    int32_t warmup_steps;       /* W: tau_h fixed and initial hot set chosen at t = W */
    int32_t dwell_min;          /* minimum steps between transitions of one expert (DESIGN.md R-C2) */
    int32_t publish_lag;        /* L: 1 <= L < Tp, transitions become stable L steps after issue (R-T1) */
    int32_t max_tokens;         /* max tokens per dx_moe_forward; sizes the workspace */
    int32_t ep_rank, ep_size;   /* expert parallelism: this GPU owns experts [r*E/G, (r+1)*E/G) */
    int32_t n_shared;           /* f-3: shared experts per layer (0 or 1, Eq. 1's first sum PAPER.md:130, R-S1): an
                                   always-on expert of every token, gate 1, kept at the HIGH tier in its own block
                                   (outside the routed experts' budget M and the controller); master pointers
                                   follow the routed ones (master[L * E_loc + l] = layer l's shared expert);
                                   tcgen05 FFN path and ep_size == 1 only */
} dx_config;

typedef struct dx_pool_s* dx_pool;

/* Derived sizes of a pool (read-only). */
typedef struct {
    int32_t  n_hot;             /* §3.5 solution (R-P2) */
    int32_t  experts_local;     /* E_loc = E / ep_size */
    int32_t  cap_hi, cap_lo;    /* blocks per tier per layer after warm-up: n_hot+s, E_loc-n_hot+s */
    int64_t  slot_bytes_hi, slot_bytes_lo; /* S_h, S_l (R-P1) */
    int64_t  layer_budget;      /* M */
    int64_t  layer_bytes;       /* bytes actually reserved per layer (<= M) */
    int64_t  arena_bytes;       /* the one device allocation */
    int64_t  export_bytes_hi, export_bytes_lo; /* dx_export_expert output sizes */
} dx_info;

/* One command of a precision plan (Alg. 1 EnqueueUpgrade/EnqueueDowngrade). */
typedef struct {
    int32_t expert;             /* local expert id */
    int32_t dir;                /* +1 promote, -1 demote, 0 relayout move (finalize only) */
    int32_t dst_slot;           /* destination block in the destination tier's region */
    int32_t src_slot;           /* block the expert occupied when the plan was made */
} dx_cmd;

#define DX_MAX_CMDS 1024
typedef struct {
    int32_t  due;               /* 1 if a plan (or the warm-up finalize) ran at this step */
    int32_t  finalize;          /* 1 at t == W: tau_h fixed, initial HIGH set installed synchronously */
    int32_t  n;                 /* number of commands */
    int64_t  step;              /* t at which the plan was made */
    int64_t  publish_step;      /* t at which the commands become the stable version */
    dx_cmd   cmd[DX_MAX_CMDS];
} dx_plan;

/* ---------------------------------------------------------------- pool lifecycle */

/* Create the slot pool of every layer (§3.4) after solving the per-layer budget
 * (§3.5).  master_bf16_host[l * E_loc + e] points to expert e's bf16 master image
 *   W_gate[I][H] | W_up[I][H] | W_down[H][I]   (row-major, nn.Linear layout, 3*I*H*2 bytes)
 * in PINNED (page-locked, UVA-mapped) host memory.  Borrowed: must outlive the pool when
 * high_bits == 16, because promotions stream HIGH images from it (the DRAM cache).
 * When high_bits < 16 the library allocates its own pinned HIGH-image cache and fills it here.
 * Every expert starts LOW in warm-up block e (R-P3).  Streams are cudaStream_t (NULL = legacy
 * default for compute; side NULL = the library creates a low-priority stream).
 * Errors: INVALID_ARG (shapes, non-pinned master), RANGE, INFEASIBLE_BUDGET, OOM, CUDA. */
dx_status dx_pool_create(const dx_config* cfg, const void* const* master_bf16_host,
                         void* compute_stream, void* side_stream, dx_pool* out);
dx_status dx_pool_destroy(dx_pool pool);
dx_status dx_pool_info(dx_pool pool, dx_info* out);

/* Expert parallelism over NCCL (north_star "partitioned across 1, 2, 4 and 8 B200s ... using NCCL
 * all-to-all"; SURVEY §8(e) collective v1).  dx_get_unique_id writes a 128-byte NCCL unique id (call on one
 * rank, broadcast it, e.g. with torch.distributed); dx_pool_create_ep is dx_pool_create plus a library-owned
 * NCCL communicator over the cfg->ep_size ranks (cfg->ep_rank = this rank; the current CUDA device is this
 * rank's GPU).  COLLECTIVE: every rank calls it with the same id and blocks until all have joined.  With a
 * communicator, dx_moe_forward / dx_moe_step run the whole expert-parallel layer inside the library:
 * dispatch over the global experts, an ncclAlltoAll of {rows per owner, token count} pairs, one device->host
 * copy of those counts (the v1 synchronisation point), grouped ncclSend/ncclRecv of the bf16 rows and
 * {local expert, gate} metadata, the owner-side FFN on the received rows (hotness counted there with B_tot =
 * the global token count, so counters and plans equal a single-GPU run on the same global batch), the return
 * exchange and the rank-order combine -- and are then collective too: every rank calls them for the same
 * layers in the same order (T may differ per rank, max_tokens may not).  ep_size = 1 with a communicator is a
 * valid loopback (self send/recv) that runs the same path on one GPU.  libnccl.so.2 is loaded at run time
 * (DX_NCCL_LIB overrides).  Errors: NCCL (library missing, init or collective failure), plus
 * dx_pool_create's.
 * f-2: the dispatch sends each token's x row ONCE per owner rank however many of its k experts that
 * rank owns, with per-entry metadata {local expert, gate, row}; results still return one row per entry.
 * nccl_id = NULL creates a member of a LOCAL group instead (several ranks' pools in one process on one device,
 * ep_rank = its index, sharing one compute stream): the same layer runs through dx_moe_step_group with the
 * exchange done by device copies. */
dx_status dx_get_unique_id(void* id128);
/* dx_moe_step for all n = ep_size pools of a local group (created with dx_pool_create_ep(nccl_id = NULL)), one
 * layer: host arrays of n entries (pool r serves x[r] [T[r]][H] -> y[r]; router_w / router_bias or logits per
 * pool).  Same results as n processes running dx_moe_step over NCCL. */
dx_status dx_moe_step_group(dx_pool* pools, int32_t n, int32_t layer, const void* const* x, const int32_t* T,
                            const void* const* router_w, const float* const* router_bias, const float* const* logits,
                            void* const* y);
/* f-2 accounting of an EP pool since creation: x rows this rank sent (deduplicated) and dispatch entries (rows an
 * undeduplicated exchange would have sent). */
dx_status dx_ep_traffic(dx_pool pool, uint64_t* rows_sent, uint64_t* entries_sent);
/* f-4 SSD tier ("stored on SSD and cached in DRAM"): dx_pool_create plus a file at ssd_path that
 * the library creates and fills with every expert's HIGH image at create time (it is removed at destroy), and a
 * pinned DRAM cache of dram_cache_images HIGH images in front of it (LRU).  Every promotion (plans, the warm-up
 * finalize, manual commands, prefetch staging) then takes its image from the cache, or reads it from the file
 * (O_DIRECT when the image size allows, so a miss really reads the device) into the least recently used slot,
 * then copies it to HBM on the copy engine.  Masters are read during create only.  ep_size 1 only. */
dx_status dx_pool_create_ssd(const dx_config* cfg, const void* const* master_bf16_host, void* compute_stream,
                             void* side_stream, const char* ssd_path, int32_t dram_cache_images, dx_pool* out);
dx_status dx_pool_create_ep(const dx_config* cfg, const void* const* master_bf16_host, void* compute_stream,
                            void* side_stream, const void* nccl_id, dx_pool* out);

/* ---------------------------------------------------------------- the MoE layer (Eq. 1) */

/* y = sum_{j in topk} g_j(x) E_j(x) (+ E^s(x) with n_shared = 1: y = bf16(E^s(x) + sum_j ...), the shared term
 * first) for T tokens of one layer, each expert
 * read at its last stable version and tier.
 *   x_bf16      [T][H] bf16, device.
 *   router_w    [E][H] bf16, device, and router_bias [E] fp32 (may be NULL): router mode,
 *               logits = x W_r^T + b in fp32 (the router stays full precision);
 *   logits      [T][E] fp32, device: trace mode (router_w must be NULL).  Exactly one of the two.
 *   y_bf16      [T][H] bf16, device (output).
 *   topk_idx    [T][k] int32 and topk_gate [T][k] fp32, device, optional outputs.
 * Also accumulates the hotness counters cnt/mass of the layer.
 * 0 <= T <= max_tokens; T = 0 is a no-op.  Asynchronous on the compute stream. */
dx_status dx_moe_forward(dx_pool pool, int32_t layer, const void* x_bf16, int32_t T,
                         const void* router_w_bf16, const float* router_bias, const float* logits,
                         void* y_bf16, int32_t* topk_idx, float* topk_gate);

/* One serving step of one layer: dx_moe_forward + dx_hotness_update + dx_plan_precision, with the EMA fold
 * and publication (a10, a14) fused into the combine launch (same results, bit for bit, as the three calls;
 * the fold runs after the layer's GEMMs so the table flip never races them).  Arguments as dx_moe_forward;
 * T = 0 folds an empty step (passive decay).  Asynchronous on the compute stream. */
dx_status dx_moe_step(dx_pool pool, int32_t layer, const void* x_bf16, int32_t T,
                      const void* router_w_bf16, const float* router_bias, const float* logits,
                      void* y_bf16, int32_t* topk_idx, float* topk_gate);

/* dx_moe_step over layers [layer0, layer0 + n_layers) in one call (a stack step without a host round trip per
 * layer): host arrays of n_layers DEVICE pointers, entry i for layer layer0 + i -- x, y, and either router_w
 * (+ router_bias, whose array may be NULL) or logits.  Entries may repeat (e.g. y ping-pong, or x[i] = y[i-1]
 * to chain the layers).  Stops at the first failing layer and returns its status. */
dx_status dx_moe_step_layers(dx_pool pool, int32_t layer0, int32_t n_layers, const void* const* x, int32_t T,
                             const void* const* router_w, const float* const* router_bias, const float* const* logits,
                             void* const* y);

/* The fp32 router logits [T][E] of the last router-mode forward of this pool (exactly what its top-k
 * consumed), into host memory of cap >= T*E floats.  Synchronising.  NOT_READY if the last forward was
 * in trace mode. */
dx_status dx_get_logits(dx_pool pool, float* host_out, int64_t cap);

/* ---------------------------------------------------------------- expert parallelism, phase by phase
 * ep_size G > 1: GPU r owns experts [r*E/G, (r+1)*E/G) (its pool holds only those, master pointers
 * [L][E/G]); tokens are data-parallel.  One layer is dispatch -> all-to-all -> owner FFN ->
 * all-to-all -> combine.  With a communicator (dx_pool_create_ep) dx_moe_forward does all of it; these
 * phase calls leave the two exchanges to the caller (used to run G pools in one process on one GPU, the
 * exchange done by device copies).  Hotness is counted on the owner from the received (expert, gate)
 * rows, so counters and plans are identical to a single-GPU run on the same global batch. */

/* Route the T local tokens over the GLOBAL experts (router mode or trace mode as dx_moe_forward) and
 * build the send buffers, rows grouped by owner rank in (t asc, j asc) order:
 *   send_rows  [T*k][H] bf16 device (x rows), send_meta [T*k] int2 device {local expert id at the owner,
 *   gate bits (fp32)}, send_counts [G] int32 device (rows per owner).  No hotness counting here. */
dx_status dx_ep_dispatch(dx_pool pool, int32_t layer, const void* x_bf16, int32_t T, const void* router_w_bf16,
                         const float* router_bias, const float* logits, void* send_rows, void* send_meta,
                         int32_t* send_counts, int32_t* topk_idx, float* topk_gate);
/* Owner side: R received rows [R][H] bf16 with their meta [R] int2; y_rows[R][H] = gate * E_e(row) for
 * the local expert e of each row (k = 1 routing given).  Accumulates the layer's hotness counters and
 * adds tokens_global (the step's global token count, B_tot of R-H2) to the fold's denominator. */
dx_status dx_moe_forward_routed(dx_pool pool, int32_t layer, const void* rows_bf16, int32_t R, const void* meta,
                                void* y_rows_bf16, int64_t tokens_global);
/* Source side: back_rows [T*k][H] bf16 are the owner results returned in dispatch order; y[T][H] =
 * bf16(sum_j back_rows[row of (t, j)]) in rank order (a8).  T must equal the last dispatch's T. */
dx_status dx_ep_combine(dx_pool pool, int32_t layer, const void* back_rows, int32_t T, void* y_bf16);

/* Fold the counters accumulated since the last fold into the EMA scores (Eq. 2, PAPER.md:226,
 * with Alg. 1's passive decay, R-H2); step t += 1; publish transitions due at the new t (R-T1).
 * Asynchronous on the compute stream (waits on the side stream only when a publish is due). */
dx_status dx_hotness_update(dx_pool pool, int32_t layer);
/* Trace mode: accumulate counters from given routing (device idx [T][k] int32 global expert ids,
 * gate [T][k] fp32; B_tot = T) and fold.  INVALID_ARG on a duplicate expert within a token. */
dx_status dx_hotness_update_from(dx_pool pool, int32_t layer, const int32_t* topk_idx,
                                 const float* topk_gate, int32_t T);

/* Alg. 1 PrecisionSchedule at the current step t of `layer`:
 *  t == W: finalize the warm-up (tau_h, initial HIGH set, synchronous relayout, R-P3);
 *  t > W, t ≡ 0 mod Tp: compute the plan on the device (R-C1..C4), reserve destination blocks and
 *  issue promotions (H2D of the HIGH image) and demotions (on-device group quantisation) on the
 *  side stream; they become stable at t + L.
 * out == NULL: fully asynchronous.  out != NULL: synchronises and reports the plan (tests). */
dx_status dx_plan_precision(dx_pool pool, int32_t layer, dx_plan* out);

/* Manual commands (EnqueueUpgrade / EnqueueDowngrade for host-chosen experts), issued like a plan.
 * Per expert: RANGE, NOT_READY (before warm-up end), INVALID_ARG (already at that tier),
 * BUSY (in flight), POOL_EXHAUSTED (no free block: deferred, nothing issued).  Synchronising. */
dx_status dx_promote(dx_pool pool, int32_t layer, const int32_t* experts, int32_t n);
dx_status dx_demote(dx_pool pool, int32_t layer, const int32_t* experts, int32_t n);

/* Wait for all compute- and side-stream work of the pool (does not move the publish schedule).
 * Reports (and clears) the sticky device error: RANGE if dx_moe_forward_routed received an expert id
 * outside [0, E_loc) since the last dx_sync (such rows were routed with gate 0, output 0). */
dx_status dx_sync(dx_pool pool);

/* ---------------------------------------------------------------- inspection (synchronising) */
dx_status dx_query_expert(dx_pool pool, int32_t layer, int32_t e, int32_t* tier, int32_t* slot,
                          uint32_t* version, int32_t* in_flight);
/* Bulk table: arrays of E_loc entries each (any may be NULL).  tier: 1 HIGH 0 LOW;
 * in_flight: +1/-1 pending direction, 0 none. */
dx_status dx_get_table(dx_pool pool, int32_t layer, int32_t* tier, int32_t* slot, uint32_t* version,
                       int32_t* in_flight);
dx_status dx_occupancy(dx_pool pool, int32_t layer, int32_t* used_hi, int32_t* cap_hi,
                       int32_t* used_lo, int32_t* cap_lo);
/* S[E_loc] fp64 scores, cnt/mass[E_loc] counters not yet folded, tau_h, n_hot, t. */
dx_status dx_get_hotness(dx_pool pool, int32_t layer, double* S, uint32_t* cnt, uint64_t* mass,
                         double* tau_h, int32_t* n_hot, int64_t* step);
/* Canonical image of expert e at its stable tier into host memory (DESIGN.md R-Q1 export):
 * bf16 tier: 3*I*H bf16 (master layout); quantised tier: codes u8 [3*I*H] unpacked | scales bf16
 * [3*I*H/g] | zeros u8 [3*I*H/g], matrices in the order gate, up, down. */
dx_status dx_export_expert(dx_pool pool, int32_t layer, int32_t e, void* host_out, int64_t cap_bytes,
                           int64_t* written);

/* ---------------------------------------------------------------- standalone group quantiser */
/* On-device group quantisation of a bf16 matrix [N][K] (row-major, groups of g along K), R-Q1:
 * codes packed little-endian along K (int4: c[k] | c[k+1]<<4; int2: 4 per byte), scales bf16
 * [N][K/g], zeros u8 [N][K/g].  All device pointers; asynchronous on `stream`. */
dx_status dx_quantize(const void* w_bf16, int64_t N, int64_t K, int32_t g, int32_t bits,
                      void* codes_packed, void* scales_bf16, void* zeros_u8, void* stream);
/* w_hat = bf16_rn((q - z) * s) into w_bf16 [N][K]. */
dx_status dx_dequantize(const void* codes_packed, const void* scales_bf16, const void* zeros_u8,
                        int64_t N, int64_t K, int32_t g, int32_t bits, void* w_bf16, void* stream);

/* Sizes in bytes of one expert slot at `bits` (R-P1), and the per-layer n_hot (R-P2); -1 if infeasible. */
int64_t dx_slot_bytes(int32_t H, int32_t I, int32_t g, int32_t bits);
int64_t dx_solve_n_hot(int64_t layer_budget, int32_t n_experts, int64_t S_h, int64_t S_l, int32_t n_spare);

/* Expert-FFN implementation: 0 = tcgen05/TMEM grouped GEMM with TMA and in-smem dequant (default),
 * 1 = register-dequant mma.sync streaming kernel (kept as an independent cross-check). */
dx_status dx_set_ffn_path(dx_pool pool, int32_t path);

/* ---------------------------------------------------------------- profiling for benches */
typedef struct {
    int64_t  forwards;          /* dx_moe_forward calls (T > 0) since the last read */
    double   fwd_ms;            /* summed device time of whole forwards (CUDA events on the compute stream) */
    double   ffn_ms[2];         /* summed device time of the gate/up (0) and down (1) expert kernels */
    uint64_t weight_bytes[2];   /* algorithmic expert-weight bytes those kernels must read: every touched
                                   expert's gate+up (0) / down (1) codes+scales+zeros at its stable tier */
    uint64_t active_experts;    /* touched experts summed over forwards */
    double   route_ms;          /* summed device time of router + top-k + placement */
    double   exposed_ms;        /* compute-stream stall waiting for side-stream transitions at publish
                                   (the exposed switch time, "never affects the forward") */
    int64_t  publishes;         /* publish points seen */
    double   xfer_ms;           /* summed side-stream duration of issued transitions (issue -> ready) */
    double   xfer_max_ms;       /* longest single plan's transitions */
    int64_t  plans;             /* plans whose transitions were issued */
    int64_t  promotions, demotions; /* transitions those plans issued */
    double   copy_ms;           /* summed side-stream time of the plans' copy-engine promotions (H2D) */
    uint64_t copy_bytes;        /* bytes those copies moved (copy_bytes / copy_ms = promotion bandwidth) */
    int64_t  prefetch_issued;   /* f-1: HIGH images staged ahead of plans */
    int64_t  prefetch_hits;     /* promotions whose image was already staged in their destination block */
    int64_t  ssd_reads;         /* f-4: HIGH images read from the SSD tier (DRAM-cache misses) */
    uint64_t ssd_bytes;
    double   ssd_read_ms;       /* host time spent in those reads */
    int64_t  dram_cache_hits;   /* HIGH images served by the DRAM cache */
    int64_t  ffn_fused;         /* profiled forwards whose FFN was ONE fused decode launch (gate/up then down):
                                   their whole FFN time is in ffn_ms[0] and ffn_ms[1] is ~0 */
} dx_profile_t;
/* f-1 cross-layer correlation prefetch.  fanout f in [0, 8] (0 = off), lead d in
 * [1, Tp - L].  With f > 0 every dx_moe_forward / dx_moe_step of layer l (the stack called layer by layer on the
 * same batch) adds, for each token, one count per pair (expert chosen at layer l-1, expert chosen at layer l) to
 * the pair's correlation matrix corr[l-1][e][e'] (u32, device, SPEC update_correlation); d steps before layer
 * l+1's next plan it scores every LOW, not-in-flight expert e' of layer l+1 by sum over layer l's current choices e
 * of corr[l][e][e'] and stages the HIGH images of the top f (score desc, id asc) into the lowest free HIGH blocks on
 * the copy engine (SPEC prefetch_candidates; the transient blocks are otherwise idle between plans).  A plan that
 * then promotes a staged expert into its staged block skips the copy (dx_profile_t prefetch_hits).  Results are
 * unchanged; only the promotion latency drops.  INVALID_ARG for EP pools. */
dx_status dx_set_prefetch(dx_pool pool, int32_t fanout, int32_t lead);
/* corr[layer][E_loc][E_loc] (the pair (layer, layer + 1)) into host memory; synchronising.  RANGE outside the stack. */
dx_status dx_get_corr(dx_pool pool, int32_t layer, uint32_t* host_out);
/* The layer's current prefetch: up to 8 {expert, HIGH block} pairs staged (or chosen and about to be) for its
 * next plan; synchronising. */
dx_status dx_get_prefetch(dx_pool pool, int32_t layer, int32_t* experts, int32_t* blocks, int32_t* n);
/* TIMING BASELINE ONLY (SURVEY §8(d) C5 "teleport"): on != 0 makes runtime plans and their publication
 * happen exactly as scheduled but skips the side-stream transfers, so the per-step tier tables are the
 * same while switching costs nothing -- and the moved experts' weights are garbage.  The exposed switch
 * time is (t_on - t_teleport) / t_on over the same steps.  Never for results. */
dx_status dx_set_teleport(dx_pool pool, int32_t on);
/* Per-forward CUDA-event timing: enable = 0 off; enable = n >= 1 times every n-th forward (n > 1 keeps the
   host cost of event records off most forwards).  While enabled, the device weight-byte counters count
   exactly the timed (sampled) forwards, so bytes / time stay consistent; while disabled they count every
   forward. */
dx_status dx_profile_enable(dx_pool pool, int32_t enable);
/* Synchronising; returns and resets the accumulated profile. */
dx_status dx_profile_read(dx_pool pool, dx_profile_t* out);

/* Number of kernels this library launched since pool creation (all streams). */
int64_t dx_kernel_launches(dx_pool pool);
const char* dx_last_error(void);
const char* dx_version(void);

#ifdef __cplusplus
}
#endif
#endif
