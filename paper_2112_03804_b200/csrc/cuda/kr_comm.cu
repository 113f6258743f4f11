// kr_comm.cu — the library's multi-GPU transport: NCCL communicators over
// the GPUs of one node (NVLink 5 / NVSwitch), one rank per GPU.
//
// The turn payoff is block diagonal over river boards, so
// the boards are sharded over the ranks and the products need no
// communication.  What crosses ranks is small and happens
// once per half-iteration (the turn solver's per-board river values) or per
// checkpoint (the per-board best-response values).  Both are ALL-GATHERS of
// per-board values followed by a fold in global board order on every rank,
// never all-reduces: the fold is the one the single-GPU solver runs, so every
// result is bitwise independent of the number of ranks.  The collectives are
// enqueued on the solver's stream and captured into its iteration graphs.
//
// Ranks come from a unique id shared by the caller (ncclCommInitRank: one
// process per GPU, e.g. under torchrun) or from one process driving a device
// list (ncclCommInitAll: krb200 solve --gpus N).
//
// NCCL is bound at run time (dlopen), not at link time: a process that also
// uses PyTorch must share PyTorch's NCCL (a second copy with the same soname
// loaded first would be picked up by libtorch and lack its symbols).  The
// library already in the process is used if there is one, else KR_NCCL_LIB
// (set by the Python package to PyTorch's bundled copy), else libnccl.so.2.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kr_common.cuh"

struct kr_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, size = 1, device = 0;
};

namespace krb {
namespace {

struct NcclApi {
    decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&::ncclCommInitRank) commInitRank = nullptr;
    decltype(&::ncclCommInitAll) commInitAll = nullptr;
    decltype(&::ncclCommDestroy) commDestroy = nullptr;
    decltype(&::ncclAllGather) allGather = nullptr;
    decltype(&::ncclGetErrorString) getErrorString = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::string err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* p = std::getenv("KR_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* f = dlsym(h, n);
            if (!f) err = std::string("NCCL lacks ") + n;
            return f;
        };
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
        api.commInitAll = reinterpret_cast<decltype(api.commInitAll)>(sym("ncclCommInitAll"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
        api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
        api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw Fail{KR_CUDA, err};
    return api;
}

}  // namespace

#define KR_NCCL(call)                                                                                \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess)                                                                       \
            throw ::krb::Fail{KR_CUDA, std::string(#call) + ": " + ::krb::nccl().getErrorString(r_)}; \
    } while (0)

void comm_allgather(kr_comm* c, const double* send, double* recv, size_t count, cudaStream_t s) {
    KR_NCCL(nccl().allGather(send, recv, count, ncclDouble, c->comm, s));
}
int comm_rank(const kr_comm* c) { return c->rank; }
int comm_size(const kr_comm* c) { return c->size; }
int comm_device(const kr_comm* c) { return c->device; }

}  // namespace krb

using krb::Fail;
using krb::guarded;

extern "C" {

int kr_comm_unique_id(uint8_t* id) {
    return guarded([&] {
        if (!id) throw Fail{KR_INVALID_INPUT, "null id buffer"};
        static_assert(sizeof(ncclUniqueId) == KR_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        KR_NCCL(krb::nccl().getUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

int kr_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, kr_comm** out) {
    return guarded([&] {
        if (!id || !out) throw Fail{KR_INVALID_INPUT, "null argument"};
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Fail{KR_INVALID_INPUT, "bad rank / size"};
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw Fail{KR_NO_DEVICE, "no CUDA device available"};
        }
        if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
        KR_CK(cudaSetDevice(device));
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* c = new kr_comm();
        c->rank = rank;
        c->size = nranks;
        c->device = device;
        const ncclResult_t r = krb::nccl().commInitRank(&c->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            throw Fail{KR_CUDA, std::string("ncclCommInitRank: ") + krb::nccl().getErrorString(r)};
        }
        *out = c;
    });
}

int kr_comm_init_all(int ndev, const int* devices, kr_comm** out) {
    return guarded([&] {
        if (ndev < 1 || !devices || !out) throw Fail{KR_INVALID_INPUT, "bad device list"};
        std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
        KR_NCCL(krb::nccl().commInitAll(comms.data(), ndev, devices));
        for (int r = 0; r < ndev; ++r) {
            auto* c = new kr_comm();
            c->comm = comms[size_t(r)];
            c->rank = r;
            c->size = ndev;
            c->device = devices[r];
            out[r] = c;
        }
    });
}

int kr_comm_destroy(kr_comm* c) {
    return guarded([&] {
        if (!c) return;
        if (c->comm) krb::nccl().commDestroy(c->comm);
        delete c;
    });
}

int kr_comm_rank(const kr_comm* c) { return c ? c->rank : -1; }
int kr_comm_size(const kr_comm* c) { return c ? c->size : 0; }

}  // extern "C"
