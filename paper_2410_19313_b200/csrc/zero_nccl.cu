// zero_nccl.cu -- the ZeRO step's collectives over NCCL for the C-ABI
// (coat_zero_step; zero.py is the torch.distributed form).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): libcoat.so keeps no
// link-time NCCL dependency, and inside a process that already loaded NCCL
// (e.g. PyTorch's) the same library instance is used.  nccl.h supplies only
// the types and enum values.
//
// Error-word agreement: the reference's step commits or throws as a whole
// (optimizer.cpp:101-114); sharded, every rank must take the decision the
// single-process step would take for the union of the shards.  The flag bits
// are spread over byte lanes, MAX-all-reduced (= OR), folded back into
// *d_flags, and -- still on the device, no host sync -- when the step must not
// change anything (NonFiniteGradient, contract NonFiniteInput) the rank's old
// weight shard is copied into the scratch the all-gather publishes.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <mutex>

#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.reduce_scatter = reinterpret_cast<decltype(a.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.reduce_scatter && a.all_gather &&
               a.all_reduce && a.error_string;
    });
    return a;
}

constexpr int kLanes = 8;   // flag bits 0..7

__global__ void flags_to_lanes_kernel(const uint32_t* flags, uint8_t* lanes) {
    if (threadIdx.x < kLanes) lanes[threadIdx.x] = uint8_t((*flags >> threadIdx.x) & 1u);
}

// lanes (MAX-reduced over ranks) -> *flags; republish the old shard when the
// step must leave everything unchanged.
__global__ void lanes_commit_kernel(const uint8_t* lanes, uint32_t* flags, const float* __restrict__ w_old,
                                    float* __restrict__ w_scratch, int64_t n) {
    uint32_t f = 0;
#pragma unroll
    for (int i = 0; i < kLanes; ++i) f |= uint32_t(lanes[i] != 0) << i;
    if (blockIdx.x == 0 && threadIdx.x == 0) *flags = f;
    if (!(f & (kFlagNonFiniteGrad | kFlagContract))) return;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        w_scratch[i] = w_old[i];
}

}  // namespace

bool nccl_available() { return api().ok; }

const char* nccl_error_string(int r) {
    return api().ok ? api().error_string(static_cast<ncclResult_t>(r)) : "NCCL library not found";
}

int nccl_unique_id(uint8_t* out128) {
    if (!api().ok) return -1;
    ncclUniqueId id;
    const ncclResult_t r = api().get_unique_id(&id);
    if (r == ncclSuccess)
        for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) out128[i] = static_cast<uint8_t>(id.internal[i]);
    return int(r);
}

int nccl_comm_init(void** comm, int nranks, const uint8_t* id128, int rank) {
    if (!api().ok) return -1;
    ncclUniqueId id;
    for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id.internal[i] = static_cast<char>(id128[i]);
    ncclComm_t c = nullptr;
    const ncclResult_t r = api().comm_init_rank(&c, nranks, id, rank);
    *comm = c;
    return int(r);
}

int nccl_comm_destroy(void* comm) {
    if (!api().ok) return -1;
    return int(api().comm_destroy(static_cast<ncclComm_t>(comm)));
}

int zero_reduce_scatter(const float* g_full, float* g_shard, int64_t n_shard, void* comm, cudaStream_t st) {
    return int(api().reduce_scatter(g_full, g_shard, size_t(n_shard), ncclFloat32, ncclSum,
                                    static_cast<ncclComm_t>(comm), st));
}

int zero_all_gather(const float* w_shard, float* w_full, int64_t n_shard, void* comm, cudaStream_t st) {
    return int(api().all_gather(w_shard, w_full, size_t(n_shard), ncclFloat32, static_cast<ncclComm_t>(comm), st));
}

// *d_flags := OR over ranks; w_scratch := w_old when nothing may change.
// `lanes` is kLanes bytes of per-call device scratch (coat_zero_step passes
// the head of its g_shard, which the fused step has consumed by then in
// stream order), so concurrent ZeRO steps -- other communicators, other
// streams on the same device -- never share it.
// Returns an NCCL result (0 = success); *cuda_err receives launch errors.
int zero_agree_and_select(uint32_t* d_flags, const float* w_old, float* w_scratch, int64_t n_shard, void* comm,
                          uint8_t* lanes, cudaStream_t st, cudaError_t* cuda_err) {
    flags_to_lanes_kernel<<<1, 32, 0, st>>>(d_flags, lanes);
    if ((*cuda_err = cudaGetLastError()) != cudaSuccess) return 0;
    const ncclResult_t r = api().all_reduce(lanes, lanes, kLanes, ncclUint8, ncclMax, static_cast<ncclComm_t>(comm), st);
    if (r != ncclSuccess) return int(r);
    const int blocks = (int)imax64(1, imin64((n_shard + 255) / 256, int64_t(device_sm_count()) * 4));
    lanes_commit_kernel<<<blocks, 256, 0, st>>>(lanes, d_flags, w_old, w_scratch, n_shard);
    *cuda_err = cudaGetLastError();
    return 0;
}

}  // namespace coat
