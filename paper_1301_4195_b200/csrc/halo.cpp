// halo.cpp -- the halo exchange of the sharded spatial domain (SPEC.md:419-481,
// PAPER.md:389-428), on NCCL over NVLink / NVSwitch.
//
// A rank owns a contiguous range of cells as a (ncl + 4) x N^3 field with two
// ghost cells per side.  Before every transport stage it sends its
// first two interior cells to the left neighbour and its last two to the right
// one, and receives the neighbours' edge cells into its ghosts.  Ghosts and edge
// cells are contiguous 2 x N^3 blocks of the field, so each direction is ONE
// message (the paper sends 4), grouped in one
// ncclGroupStart/End so there is no even/odd ordering.
// Physical-end ghosts (wall / extrapolation) stay local (boltz_fill_boundary).
//
// Communicators: one process per GPU (boltz_halo_unique_id on rank 0, shared
// out of band, then boltz_halo_create on every rank) or one process driving
// several GPUs (boltz_halo_create_all, ncclCommInitAll).  The in-process
// loopback backend copies ghosts between per-rank fields of one
// device without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/boltz_cuda.h"

namespace boltz_gpu {
void set_error(const std::string& s);  // boltz_cuda.cu (thread-local, boltz_last_error)
}

struct boltz_halo {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};

namespace {

// NCCL is bound lazily with dlopen on the first halo call, so the library has
// no link-time NCCL dependency.  Order: $BOLTZ_NCCL_LIB, else a libnccl.so.2
// the process already loaded (e.g. PyTorch's; RTLD_NOLOAD), else the system
// one.  A process that uses PyTorch too must import it BEFORE the first halo
// call: a later torch import would otherwise find the system NCCL under its
// soname.
struct Nccl {
    decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&::ncclCommInitRank) CommInitRank = nullptr;
    decltype(&::ncclCommInitAll) CommInitAll = nullptr;
    decltype(&::ncclCommDestroy) CommDestroy = nullptr;
    decltype(&::ncclGroupStart) GroupStart = nullptr;
    decltype(&::ncclGroupEnd) GroupEnd = nullptr;
    decltype(&::ncclSend) Send = nullptr;
    decltype(&::ncclRecv) Recv = nullptr;
    decltype(&::ncclAllReduce) AllReduce = nullptr;
    decltype(&::ncclGetErrorString) GetErrorString = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (const char* path = std::getenv("BOLTZ_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        bool all = true;
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            all = all && fp != nullptr;
        };
        sym(n.GetUniqueId, "ncclGetUniqueId");
        sym(n.CommInitRank, "ncclCommInitRank");
        sym(n.CommInitAll, "ncclCommInitAll");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
        sym(n.AllReduce, "ncclAllReduce");
        sym(n.GetErrorString, "ncclGetErrorString");
        n.ok = all;
    });
    return n;
}

#define NCCL_OR_FAIL()                                                      \
    do {                                                                    \
        if (!nccl().ok) {                                                   \
            boltz_gpu::set_error("NCCL (libnccl.so.2) could not be loaded"); \
            return BOLTZ_ERR_CUDA;                                          \
        }                                                                   \
    } while (0)

int nccl_fail(const char* what, ncclResult_t r) {
    boltz_gpu::set_error(std::string(what) + ": " + nccl().GetErrorString(r));
    return BOLTZ_ERR_CUDA;
}

int cuda_fail(const char* what, cudaError_t e) {
    boltz_gpu::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return BOLTZ_ERR_CUDA;
}

}  // namespace

extern "C" {

int boltz_halo_unique_id(unsigned char id[BOLTZ_HALO_ID_BYTES]) {
    NCCL_OR_FAIL();
    if (!id) {
        boltz_gpu::set_error("halo_unique_id: null output");
        return BOLTZ_ERR_CONFIG;
    }
    ncclUniqueId u;
    if (ncclResult_t r = nccl().GetUniqueId(&u); r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    static_assert(sizeof(u.internal) == BOLTZ_HALO_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, u.internal, BOLTZ_HALO_ID_BYTES);
    return BOLTZ_OK;
}

int boltz_halo_create(int rank, int world, const unsigned char id[BOLTZ_HALO_ID_BYTES], int device,
                      boltz_halo** out) {
    NCCL_OR_FAIL();
    if (!out || !id || world < 1 || rank < 0 || rank >= world) {
        boltz_gpu::set_error("halo_create: need 0 <= rank < world, an id and an output pointer");
        return BOLTZ_ERR_CONFIG;
    }
    if (cudaError_t e = cudaSetDevice(device); e != cudaSuccess) return cuda_fail("cudaSetDevice", e);
    ncclUniqueId u;
    std::memcpy(u.internal, id, BOLTZ_HALO_ID_BYTES);
    auto* h = new boltz_halo();
    h->rank = rank;
    h->world = world;
    h->device = device;
    if (ncclResult_t r = nccl().CommInitRank(&h->comm, world, u, rank); r != ncclSuccess) {
        delete h;
        return nccl_fail("ncclCommInitRank", r);
    }
    *out = h;
    return BOLTZ_OK;
}

int boltz_halo_create_all(int world, const int* devices, boltz_halo** out) {
    NCCL_OR_FAIL();
    if (world < 1 || !devices || !out) {
        boltz_gpu::set_error("halo_create_all: need world >= 1, devices[world] and out[world]");
        return BOLTZ_ERR_CONFIG;
    }
    std::vector<ncclComm_t> comms(world);
    if (ncclResult_t r = nccl().CommInitAll(comms.data(), world, devices); r != ncclSuccess)
        return nccl_fail("ncclCommInitAll", r);
    for (int i = 0; i < world; ++i) {
        out[i] = new boltz_halo();
        out[i]->comm = comms[i];
        out[i]->rank = i;
        out[i]->world = world;
        out[i]->device = devices[i];
    }
    return BOLTZ_OK;
}

int boltz_halo_destroy(boltz_halo* h) {
    if (!h) return BOLTZ_OK;
    if (!nccl().ok) {
        delete h;
        return BOLTZ_OK;
    }
    ncclResult_t r = h->comm ? nccl().CommDestroy(h->comm) : ncclSuccess;
    delete h;
    return r == ncclSuccess ? BOLTZ_OK : nccl_fail("ncclCommDestroy", r);
}

int boltz_halo_exchange(boltz_halo* h, double* field, int64_t ncl, int64_t n3, void* stream) {
    NCCL_OR_FAIL();
    if (!h || !field || ncl < 2 || n3 < 1) {
        boltz_gpu::set_error("halo_exchange: need a halo, a field and >= 2 interior cells");
        return BOLTZ_ERR_CONFIG;
    }
    if (cudaError_t e = cudaSetDevice(h->device); e != cudaSuccess) return cuda_fail("cudaSetDevice", e);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t blk = 2 * (size_t)n3;  // two cells per direction, contiguous
    ncclResult_t r = nccl().GroupStart();
    if (r == ncclSuccess && h->rank > 0) {
        r = nccl().Send(field + 2 * n3, blk, ncclDouble, h->rank - 1, h->comm, s);                      // first two interior
        if (r == ncclSuccess) r = nccl().Recv(field, blk, ncclDouble, h->rank - 1, h->comm, s);          // left ghosts
    }
    if (r == ncclSuccess && h->rank < h->world - 1) {
        r = nccl().Send(field + (size_t)ncl * n3, blk, ncclDouble, h->rank + 1, h->comm, s);            // last two interior
        if (r == ncclSuccess) r = nccl().Recv(field + (size_t)(ncl + 2) * n3, blk, ncclDouble, h->rank + 1, h->comm, s);
    }
    ncclResult_t r2 = nccl().GroupEnd();
    if (r != ncclSuccess) return nccl_fail("halo_exchange", r);
    if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
    return BOLTZ_OK;
}

int boltz_halo_allreduce_sum(boltz_halo* h, double* buf, int64_t count, void* stream) {
    NCCL_OR_FAIL();
    if (!h || !buf || count < 0) {
        boltz_gpu::set_error("halo_allreduce_sum: invalid arguments");
        return BOLTZ_ERR_CONFIG;
    }
    if (cudaError_t e = cudaSetDevice(h->device); e != cudaSuccess) return cuda_fail("cudaSetDevice", e);
    if (ncclResult_t r = nccl().AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, h->comm, (cudaStream_t)stream);
        r != ncclSuccess)
        return nccl_fail("ncclAllReduce", r);
    return BOLTZ_OK;
}

int boltz_halo_exchange_loopback(double* const* fields, const int64_t* ncl, int nranks, int64_t n3, void* stream) {
    if (!fields || !ncl || nranks < 1 || n3 < 1) {
        boltz_gpu::set_error("halo_exchange_loopback: invalid arguments");
        return BOLTZ_ERR_CONFIG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = 2 * (size_t)n3 * sizeof(double);
    for (int r = 0; r + 1 < nranks; ++r) {
        if (ncl[r] < 2 || ncl[r + 1] < 2) {
            boltz_gpu::set_error("halo_exchange_loopback: every rank needs >= 2 interior cells");
            return BOLTZ_ERR_CONFIG;
        }
        double* a = fields[r];
        double* b = fields[r + 1];
        // right ghosts of r <- first two interior of r+1; left ghosts of r+1 <- last two interior of r
        if (cudaError_t e = cudaMemcpyAsync(a + (size_t)(ncl[r] + 2) * n3, b + 2 * n3, bytes, cudaMemcpyDeviceToDevice, s);
            e != cudaSuccess)
            return cuda_fail("halo_exchange_loopback", e);
        if (cudaError_t e = cudaMemcpyAsync(b, a + (size_t)ncl[r] * n3, bytes, cudaMemcpyDeviceToDevice, s);
            e != cudaSuccess)
            return cuda_fail("halo_exchange_loopback", e);
    }
    return BOLTZ_OK;
}

}  // extern "C"
