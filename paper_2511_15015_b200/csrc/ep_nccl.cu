// ep_nccl.cu -- the NCCL transport of expert parallelism (SURVEY §8(e) "collective v1"; north_star "experts are
// partitioned across 1, 2, 4 and 8 B200s ... using NCCL all-to-all").  One process per GPU; GPU r owns experts
// [r*E/G, (r+1)*E/G).  Per layer the library exchanges, on the pool's compute stream:
//   1. ncclAlltoAll (grouped send/recv before NCCL 2.28) of {rows for peer d, my token count} pairs (G x 2 int32),
//      then ONE device->host copy of the send and receive counts (the v1 host synchronisation: the grouped
//      send/recv below need the sizes);
//   2. grouped ncclSend/ncclRecv of the dispatched bf16 rows and their {local expert, gate} metadata;
//   3. after the owner-side FFN, the mirror-image grouped send/recv of the result rows.
// libnccl is loaded at run time (dlopen): the process normally already holds torch's NCCL 2.28
// (nvidia/nccl/lib/libnccl.so.2); DX_NCCL_LIB names another build.  No NCCL type crosses the C ABI.
#include "dx_common.cuh"
#include <dlfcn.h>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace {

typedef int nres_t;                    // ncclResult_t (0 = ncclSuccess)
typedef void* ncomm_t;                 // ncclComm_t
struct NId { char b[128]; };           // ncclUniqueId
enum { NCCL_INT32 = 2, NCCL_UINT8 = 1, NCCL_BF16 = 9 };   // ncclInt32, ncclUint8, ncclBfloat16 (nccl.h 2.28)

struct NcclApi {
    nres_t (*GetUniqueId)(NId*) = nullptr;
    nres_t (*CommInitRank)(ncomm_t*, int, NId, int) = nullptr;
    nres_t (*CommDestroy)(ncomm_t) = nullptr;
    nres_t (*AlltoAll)(const void*, void*, size_t, int, ncomm_t, cudaStream_t) = nullptr;
    nres_t (*Send)(const void*, size_t, int, int, ncomm_t, cudaStream_t) = nullptr;
    nres_t (*Recv)(void*, size_t, int, int, ncomm_t, cudaStream_t) = nullptr;
    nres_t (*GroupStart)() = nullptr;
    nres_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(nres_t) = nullptr;
    nres_t (*GetVersion)(int*) = nullptr;
    bool ok = false;
    char why[256] = "";
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {getenv("DX_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* n : names) {
            if (!n || !*n) continue;
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            snprintf(a.why, sizeof(a.why), "dlopen(libnccl.so.2) failed: %s", dlerror());
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                ok = false;
                snprintf(a.why, sizeof(a.why), "libnccl lacks %s", name);
            }
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        a.AlltoAll = reinterpret_cast<decltype(a.AlltoAll)>(dlsym(h, "ncclAlltoAll"));   // 2.28+; else send/recv
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        sym(a.GetVersion, "ncclGetVersion");
        a.ok = ok;
    });
    return a;
}

dx_status nfail(const char* what, nres_t r) {
    dx_set_error("%s failed: %s (nccl %d)", what, api().GetErrorString ? api().GetErrorString(r) : "?", r);
    return DX_ERR_NCCL;
}

}  // namespace

#define NCHECK(call, what)                       \
    do {                                         \
        const nres_t r_ = (call);                \
        if (r_ != 0) return nfail(what, r_);     \
    } while (0)

dx_status ep_nccl_available() {
    NcclApi& a = api();
    if (!a.ok) {
        dx_set_error("NCCL unavailable: %s", a.why);
        return DX_ERR_NCCL;
    }
    return DX_OK;
}

int ep_nccl_version() {
    int v = 0;
    if (api().ok) api().GetVersion(&v);
    return v;
}

dx_status ep_nccl_unique_id(void* id128) {
    dx_status st = ep_nccl_available();
    if (st != DX_OK) return st;
    NId id;
    NCHECK(api().GetUniqueId(&id), "ncclGetUniqueId");
    memcpy(id128, &id, sizeof(id));
    return DX_OK;
}

// collective over the G ranks: every rank calls it with the same id (blocking until all joined)
dx_status ep_nccl_init(const void* id128, int G, int rank, void** comm) {
    dx_status st = ep_nccl_available();
    if (st != DX_OK) return st;
    NId id;
    memcpy(&id, id128, sizeof(id));
    ncomm_t c = nullptr;
    NCHECK(api().CommInitRank(&c, G, id, rank), "ncclCommInitRank");
    *comm = c;
    return DX_OK;
}

void ep_nccl_destroy(void* comm) {
    if (comm && api().ok) api().CommDestroy(comm);
}

// per-peer count tuples of `per` int32: tup[d] for peer d -> recv_tup[s] from peer s
dx_status ep_nccl_exchange_counts(void* comm, int G, int per, const int32_t* tup, int32_t* recv_tup, cudaStream_t st) {
    NcclApi& a = api();
    if (a.AlltoAll) {
        NCHECK(a.AlltoAll(tup, recv_tup, (size_t)per, NCCL_INT32, comm, st), "ncclAlltoAll(counts)");
        return DX_OK;
    }
    NCHECK(a.GroupStart(), "ncclGroupStart");               // NCCL < 2.28: the same exchange as grouped send/recv
    for (int p = 0; p < G; ++p) {
        NCHECK(a.Send(tup + per * p, (size_t)per, NCCL_INT32, p, comm, st), "ncclSend(counts)");
        NCHECK(a.Recv(recv_tup + per * p, (size_t)per, NCCL_INT32, p, comm, st), "ncclRecv(counts)");
    }
    NCHECK(a.GroupEnd(), "ncclGroupEnd");
    return DX_OK;
}

// rows of H bf16 (block for peer p: [soff[p], soff[p] + sc[p]) out, [roff[p], roff[p] + rc[p]) in) and, when
// send_meta != NULL, `mi` int32 of metadata per entry with separate entry counts/offsets (se/seoff, re/reoff: with
// deduplicated rows a peer gets fewer rows than entries)
dx_status ep_nccl_exchange_rows(void* comm, int G, int H, const void* send_rows, const int* sc, const int* soff,
                                void* recv_rows, const int* rc, const int* roff, const void* send_meta, const int* se,
                                const int* seoff, void* recv_meta, const int* re, const int* reoff, int mi,
                                cudaStream_t st) {
    NcclApi& a = api();
    const size_t rb = (size_t)H * 2;
    NCHECK(a.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < G; ++p) {
        if (sc[p] > 0)
            NCHECK(a.Send(static_cast<const uint8_t*>(send_rows) + (size_t)soff[p] * rb, (size_t)sc[p] * H, NCCL_BF16, p,
                          comm, st), "ncclSend(rows)");
        if (send_meta && se[p] > 0)
            NCHECK(a.Send(static_cast<const int32_t*>(send_meta) + (size_t)seoff[p] * mi, (size_t)se[p] * mi, NCCL_INT32,
                          p, comm, st), "ncclSend(meta)");
        if (rc[p] > 0)
            NCHECK(a.Recv(static_cast<uint8_t*>(recv_rows) + (size_t)roff[p] * rb, (size_t)rc[p] * H, NCCL_BF16, p, comm,
                          st), "ncclRecv(rows)");
        if (recv_meta && re[p] > 0)
            NCHECK(a.Recv(static_cast<int32_t*>(recv_meta) + (size_t)reoff[p] * mi, (size_t)re[p] * mi, NCCL_INT32, p,
                          comm, st), "ncclRecv(meta)");
    }
    NCHECK(a.GroupEnd(), "ncclGroupEnd");
    return DX_OK;
}
