// NCCL over NVLink/NVSwitch for the K-sharded REINFORCE step.
//
// The reference has no collective: its K placements are evaluated by threads of
// one process (pkg/trainer.py:269-280).  Sharding K across GPUs needs exactly
// two exchanges per update (paper_1706_04972_b200/parallel.py): an all-gather
// of the per-sample scores (+ each rank's best candidate row) and a sum
// all-reduce of the fp64 policy gradient.  This file binds NCCL directly so
// that
//   * one process can drive every GPU of the box (ncclCommInitAll: a plain
//     train() call uses all visible devices), and
//   * the collectives are enqueued on the controller's stream and captured in
//     its CUDA graph together with the kernels (NCCL >= 2.9 is
//     stream-capturable), one graph replay per update at any world size.
// libnccl is opened with dlopen (the torch-bundled libnccl.so.2 is already
// resident when torch is imported), so the library loads without NCCL and the
// entry points report DP_ECOMM when it is absent.

#include <dlfcn.h>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace {

using nccl_result_t = int;
struct nccl_uid {
    char internal[128];
};
using nccl_comm_t = void *;
// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int kNcclUint8 = 1, kNcclFloat64 = 8;
constexpr int kNcclSum = 0, kNcclMin = 3;

struct NcclApi {
    bool loaded = false;
    nccl_result_t (*GetVersion)(int *) = nullptr;
    nccl_result_t (*GetUniqueId)(nccl_uid *) = nullptr;
    nccl_result_t (*CommInitRank)(nccl_comm_t *, int, nccl_uid, int) = nullptr;
    nccl_result_t (*CommInitAll)(nccl_comm_t *, int, const int *) = nullptr;
    nccl_result_t (*CommDestroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*AllGather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*GroupStart)() = nullptr;
    nccl_result_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(nccl_result_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.loaded) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    auto sym = [&](auto &fn, const char *name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        return fn != nullptr;
    };
    bool ok = sym(g_nccl.GetVersion, "ncclGetVersion") && sym(g_nccl.GetUniqueId, "ncclGetUniqueId") &&
              sym(g_nccl.CommInitRank, "ncclCommInitRank") && sym(g_nccl.CommInitAll, "ncclCommInitAll") &&
              sym(g_nccl.CommDestroy, "ncclCommDestroy") && sym(g_nccl.AllReduce, "ncclAllReduce") &&
              sym(g_nccl.AllGather, "ncclAllGather") && sym(g_nccl.GroupStart, "ncclGroupStart") &&
              sym(g_nccl.GroupEnd, "ncclGroupEnd") && sym(g_nccl.GetErrorString, "ncclGetErrorString");
    g_nccl.loaded = ok;
    return ok;
}

}  // namespace

struct dp_comm {
    nccl_comm_t comm;
    int nranks, rank, device;
};

#define DP_NCCL_TRY(call)                                                                           \
    do {                                                                                            \
        const nccl_result_t r_ = (call);                                                            \
        if (r_ != 0) {                                                                              \
            dp::set_error(std::string("NCCL: ") + #call + ": " + g_nccl.GetErrorString(r_));        \
            return DP_ECOMM;                                                                        \
        }                                                                                           \
    } while (0)

#define DP_NCCL_REQUIRE_LOADED()                                                                     \
    do {                                                                                            \
        if (!nccl_load()) {                                                                         \
            dp::set_error("NCCL: libnccl.so.2 could not be opened (dlopen)");                       \
            return DP_ECOMM;                                                                        \
        }                                                                                           \
    } while (0)

extern "C" int dp_comm_version(int32_t *version) {
    DP_ENTRY();
    DP_REQUIRE(version, "dp_comm_version: NULL argument");
    DP_NCCL_REQUIRE_LOADED();
    int v = 0;
    DP_NCCL_TRY(g_nccl.GetVersion(&v));
    *version = v;
    return DP_OK;
}

extern "C" int dp_comm_unique_id(uint8_t *id_out) {
    DP_ENTRY();
    DP_REQUIRE(id_out, "dp_comm_unique_id: NULL argument");
    DP_NCCL_REQUIRE_LOADED();
    nccl_uid id;
    DP_NCCL_TRY(g_nccl.GetUniqueId(&id));
    memcpy(id_out, id.internal, sizeof(id.internal));
    return DP_OK;
}

extern "C" int dp_comm_init_rank(int32_t nranks, const uint8_t *id, int32_t rank, dp_comm **out) {
    DP_ENTRY();
    DP_REQUIRE(id && out && nranks >= 1 && rank >= 0 && rank < nranks, "dp_comm_init_rank: bad argument");
    DP_NCCL_REQUIRE_LOADED();
    nccl_uid uid;
    memcpy(uid.internal, id, sizeof(uid.internal));
    int dev = 0;
    DP_CUDA_TRY(cudaGetDevice(&dev));
    nccl_comm_t c = nullptr;
    DP_NCCL_TRY(g_nccl.CommInitRank(&c, nranks, uid, rank));
    *out = new dp_comm{c, nranks, rank, dev};
    return DP_OK;
}

extern "C" int dp_comm_init_all(int32_t ndev, const int32_t *devices, dp_comm **out) {
    DP_ENTRY();
    DP_REQUIRE(ndev >= 1 && devices && out, "dp_comm_init_all: bad argument");
    DP_NCCL_REQUIRE_LOADED();
    std::vector<nccl_comm_t> cs(ndev, nullptr);
    std::vector<int> devs(devices, devices + ndev);
    DP_NCCL_TRY(g_nccl.CommInitAll(cs.data(), ndev, devs.data()));
    for (int i = 0; i < ndev; i++) out[i] = new dp_comm{cs[i], ndev, i, devs[i]};
    return DP_OK;
}

extern "C" void dp_comm_destroy(dp_comm *c) {
    if (!c) return;
    if (g_nccl.loaded && c->comm) g_nccl.CommDestroy(c->comm);
    delete c;
}

extern "C" int dp_comm_group_start(void) {
    DP_ENTRY();
    DP_NCCL_REQUIRE_LOADED();
    DP_NCCL_TRY(g_nccl.GroupStart());
    return DP_OK;
}

extern "C" int dp_comm_group_end(void) {
    DP_ENTRY();
    DP_NCCL_REQUIRE_LOADED();
    DP_NCCL_TRY(g_nccl.GroupEnd());
    return DP_OK;
}

extern "C" int dp_comm_all_gather(dp_comm *c, const void *send, void *recv, int64_t bytes_per_rank, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(c && send && recv && bytes_per_rank >= 0, "dp_comm_all_gather: bad argument");
    DP_NCCL_REQUIRE_LOADED();
    DP_NCCL_TRY(g_nccl.AllGather(send, recv, (size_t)bytes_per_rank, kNcclUint8, c->comm, (cudaStream_t)stream));
    return DP_OK;
}

extern "C" int dp_comm_all_reduce_f64(dp_comm *c, double *buf, int64_t count, int32_t op_min, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(c && buf && count >= 0, "dp_comm_all_reduce_f64: bad argument");
    DP_NCCL_REQUIRE_LOADED();
    DP_NCCL_TRY(g_nccl.AllReduce(buf, buf, (size_t)count, kNcclFloat64, op_min ? kNcclMin : kNcclSum, c->comm,
                                 (cudaStream_t)stream));
    return DP_OK;
}
