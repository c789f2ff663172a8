// comm.cu - one long number sharded by limb range across GPUs, driven from C++ (config 5
// at G > 1; SURVEY.md §8(b) dotg_add_words_sharded, §8(e) steps 1-5).
//
// The reference has no distribution: its long number is one serial chain of w-limb
// chunks (/root/reference/proj/src/addsub.cpp:147-164, run_words 136-170), each chunk's
// carry-in the previous chunk's carry-out. Here each rank owns a contiguous limb range
// and the chain between ranks collapses to ONE 8-byte exchange of shard aggregates:
//   1. launch_long_local  - the shard's streaming pass with an unknown carry-in X; every
//                           limb that does not depend on X is written, plus {G, P}
//   2. ncclAllGather      - {G_r, P_r} of every rank (uint32[2] per rank), on `stream`
//   3. launch_long_finish - X_r = exclusive (G, P) scan over lower ranks on the device,
//                           boundary fix-up of the shard's deferred leading run
// All three are enqueued on the caller's stream: no host synchronisation, capturable.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): inside a PyTorch process that is
// the NCCL torch already loaded (one copy per process), elsewhere the system library. A
// missing NCCL surfaces as DOTG_ENCCL from the comm entry points only; nothing else in
// the library depends on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dotg.h"
#include "internal.h"

struct dotg_comm {
    ncclComm_t nccl;
    int rank, world, device;
    bool owned;  // created by dotg_comm_init_rank (destroyed with the dotg_comm)
};

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*cu_device)(const ncclComm_t, int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* override_path = std::getenv("DOTG_NCCL_LIB");
        void* h = nullptr;
        if (override_path) {
            h = dlopen(override_path, RTLD_NOW | RTLD_GLOBAL);
        } else {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) {
            const char* e = dlerror();
            api.load_error = std::string("cannot load NCCL: ") + (e ? e : "unknown");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(sym("ncclCommInitRank"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.count = reinterpret_cast<decltype(api.count)>(sym("ncclCommCount"));
        api.user_rank = reinterpret_cast<decltype(api.user_rank)>(sym("ncclCommUserRank"));
        api.cu_device = reinterpret_cast<decltype(api.cu_device)>(sym("ncclCommCuDevice"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = api.get_unique_id && api.init_rank && api.destroy && api.all_gather && api.count && api.user_rank &&
                 api.cu_device && api.error_string;
        if (!api.ok) api.load_error = "NCCL library lacks a required symbol";
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
    const NcclApi& n = nccl();
    return dotg::api_fail(DOTG_ENCCL, std::string(where) + ": " + (n.error_string ? n.error_string(r) : "nccl error"));
}

int need_nccl() {
    const NcclApi& n = nccl();
    return n.ok ? DOTG_OK : dotg::api_fail(DOTG_ENCCL, n.load_error);
}

int words_sharded(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, uint32_t* carry_out,
                  const dotg_comm* comm, cudaStream_t st) {
    if (comm == nullptr) return dotg::api_fail(DOTG_EINVAL, "sharded: null comm");
    int rc = dotg::api_check_addsub_words(out, a, b, m);
    if (rc != DOTG_OK) return rc;
    if ((rc = dotg::api_check_device()) != DOTG_OK) return rc;
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != comm->device)
        return dotg::api_fail(DOTG_EINVAL, "sharded: current device differs from the communicator's device");
    const NcclApi& n = nccl();
    // scratch: tile state of the shard, its aggregate, the gathered aggregates, a dummy
    // carry word for m == 0 shards (they still take part in the exchange)
    const size_t sb = (dotg::long_state_bytes(m > 0 ? m : 1) + 255) / 256 * 256;
    const size_t bytes = sb + 256 + size_t(comm->world) * 8;
    char* base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), bytes, st);
    if (e != cudaSuccess) return dotg::api_fail(DOTG_ENOMEM, std::string("sharded scratch: ") + cudaGetErrorString(e));
    void* state = base;
    uint32_t* agg = reinterpret_cast<uint32_t*>(base + sb);
    uint32_t* all = reinterpret_cast<uint32_t*>(base + sb + 256);
    // an empty shard is all-propagate with no generate: {G, P} = {0, 1}
    if (m == 0) {
        e = dotg::launch_shard_identity(agg, st);
    } else {
        e = dotg::launch_long_local(sub, out, a, b, m, state, agg, st);
    }
    if (e != cudaSuccess) {
        cudaFreeAsync(base, st);
        return dotg::api_fail(DOTG_ECUDA, std::string("sharded local pass: ") + cudaGetErrorString(e));
    }
    const ncclResult_t r = n.all_gather(agg, all, 2, ncclUint32, comm->nccl, st);
    if (r != ncclSuccess) {
        cudaFreeAsync(base, st);
        return nccl_fail(r, "sharded exchange (ncclAllGather)");
    }
    if (m > 0) {
        e = dotg::launch_long_finish(sub, out, m, state, all, comm->rank, comm->world, carry_out, st);
    } else if (carry_out != nullptr) {
        // the whole-number carry still has to come out of an empty shard: compose all ranks
        e = dotg::launch_compose_aggs(all, comm->world, carry_out, st);
    }
    cudaError_t e2 = cudaFreeAsync(base, st);
    if (e != cudaSuccess) return dotg::api_fail(DOTG_ECUDA, std::string("sharded finish: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess) return dotg::api_fail(DOTG_ECUDA, std::string("sharded free: ") + cudaGetErrorString(e2));
    return DOTG_OK;
}

}  // namespace

extern "C" {

size_t dotg_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

int dotg_comm_get_unique_id(void* id) {
    if (id == nullptr) return dotg::api_fail(DOTG_EINVAL, "comm: null id buffer");
    int rc = need_nccl();
    if (rc != DOTG_OK) return rc;
    ncclUniqueId u;
    const ncclResult_t r = nccl().get_unique_id(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return DOTG_OK;
}

int dotg_comm_init_rank(dotg_comm** comm, int world, const void* id, int rank) {
    if (comm == nullptr || id == nullptr) return dotg::api_fail(DOTG_EINVAL, "comm init: null argument");
    *comm = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return dotg::api_fail(DOTG_EINVAL, "comm init: bad rank/world");
    int rc = need_nccl();
    if (rc != DOTG_OK) return rc;
    if ((rc = dotg::api_check_device()) != DOTG_OK) return rc;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    const ncclResult_t r = nccl().init_rank(&c, world, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    int dev = -1;
    cudaGetDevice(&dev);
    *comm = new dotg_comm{c, rank, world, dev, true};
    return DOTG_OK;
}

int dotg_comm_wrap(dotg_comm** comm, void* nccl_comm) {
    if (comm == nullptr || nccl_comm == nullptr) return dotg::api_fail(DOTG_EINVAL, "comm wrap: null argument");
    *comm = nullptr;
    int rc = need_nccl();
    if (rc != DOTG_OK) return rc;
    const NcclApi& n = nccl();
    ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
    int world = 0, rank = 0, dev = -1;
    ncclResult_t r = n.count(c, &world);
    if (r == ncclSuccess) r = n.user_rank(c, &rank);
    if (r == ncclSuccess) r = n.cu_device(c, &dev);
    if (r != ncclSuccess) return nccl_fail(r, "comm wrap");
    *comm = new dotg_comm{c, rank, world, dev, false};
    return DOTG_OK;
}

int dotg_comm_destroy(dotg_comm* comm) {
    if (comm == nullptr) return DOTG_OK;
    int rc = DOTG_OK;
    if (comm->owned) {
        const ncclResult_t r = nccl().destroy(comm->nccl);
        if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommDestroy");
    }
    delete comm;
    return rc;
}

int dotg_comm_rank(const dotg_comm* comm) { return comm ? comm->rank : -1; }
int dotg_comm_size(const dotg_comm* comm) { return comm ? comm->world : -1; }

int dotg_add_words_sharded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m_local, uint32_t* carry_out,
                           const dotg_comm* comm, dotg_stream_t stream) {
    return words_sharded(false, out, a, b, m_local, carry_out, comm, static_cast<cudaStream_t>(stream));
}

int dotg_sub_words_sharded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m_local, uint32_t* carry_out,
                           const dotg_comm* comm, dotg_stream_t stream) {
    return words_sharded(true, out, a, b, m_local, carry_out, comm, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
