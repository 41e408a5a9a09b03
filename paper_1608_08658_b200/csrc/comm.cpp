// Ghost-plane exchange between z-slab ranks over NCCL point-to-point
// (NVLink 5 / NVSwitch on a B200 node).  The reference has no distributed
// path; this is the build's multi-GPU row.
//
// NCCL is loaded at run time (the copy PyTorch ships, or SFDB200_NCCL_LIB) so
// the library has no link-time NCCL dependency; the communicator is created
// from a unique id the caller distributes (torch.distributed in bench.py).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "plan.hpp"

namespace sfdb200 {
namespace {

// The stable subset of nccl.h this file needs.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int ncclFloat32 = 7;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
    static Nccl n = [] {
        const char* cands[] = {std::getenv("SFDB200_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* c : cands)
            if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) fail(SFDB200_ECUDA, "NCCL (libnccl.so.2) could not be loaded; set SFDB200_NCCL_LIB");
        Nccl f{};
        auto sym = [&](const char* name) {
            void* s = dlsym(h, name);
            if (!s) fail(SFDB200_ECUDA, std::string("NCCL symbol missing: ") + name);
            return s;
        };
        f.GetUniqueId = reinterpret_cast<decltype(f.GetUniqueId)>(sym("ncclGetUniqueId"));
        f.CommInitRank = reinterpret_cast<decltype(f.CommInitRank)>(sym("ncclCommInitRank"));
        f.CommDestroy = reinterpret_cast<decltype(f.CommDestroy)>(sym("ncclCommDestroy"));
        f.Send = reinterpret_cast<decltype(f.Send)>(sym("ncclSend"));
        f.Recv = reinterpret_cast<decltype(f.Recv)>(sym("ncclRecv"));
        f.GroupStart = reinterpret_cast<decltype(f.GroupStart)>(sym("ncclGroupStart"));
        f.GroupEnd = reinterpret_cast<decltype(f.GroupEnd)>(sym("ncclGroupEnd"));
        f.GetErrorString =
            reinterpret_cast<decltype(f.GetErrorString)>(sym("ncclGetErrorString"));
        return f;
    }();
    return n;
}

void nck(ncclResult_t r, const char* what) {
    if (r != 0) fail(SFDB200_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

struct Comm {
    ncclComm_t nc = nullptr;
    int world = 1, rank = 0, device = 0;
    bool loopback = false;
};

Comm* comm_create_loopback(int world, int rank, int device) {
    if (world < 1 || rank < 0 || rank >= world) fail(SFDB200_EINVAL, "bad rank / world size");
    auto* c = new Comm;
    c->world = world;
    c->rank = rank;
    c->device = device;
    c->loopback = true;
    return c;
}

bool comm_loopback(const Comm* c) { return c && c->loopback; }

void comm_unique_id(void* id128) {
    ncclUniqueId id;
    nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof id);
}

Comm* comm_create(const void* id128, int world, int rank, int device) {
    if (world < 1 || rank < 0 || rank >= world) fail(SFDB200_EINVAL, "bad rank / world size");
    auto* c = new Comm;
    c->world = world;
    c->rank = rank;
    c->device = device;
    if (world > 1) {
        ck(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        const ncclResult_t r = nccl().CommInitRank(&c->nc, world, id, rank);
        if (r != 0) {
            delete c;
            nck(r, "ncclCommInitRank");
        }
    }
    return c;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->nc) nccl().CommDestroy(c->nc);
    delete c;
}

int comm_world(const Comm* c) { return c ? c->world : 1; }
int comm_rank(const Comm* c) { return c ? c->rank : 0; }
int comm_device(const Comm* c) { return c ? c->device : 0; }

// Rank r sends its first R updated planes to r-1 (they are r-1's bottom
// ghosts) and its last R to r+1, and receives its own ghosts; one NCCL group.
void comm_exchange(Comm* c, sfdb200_plan& p, float* row, cudaStream_t s) {
    if (!c || c->world == 1 || c->loopback) return;
    const FieldGeom& g = p.g;
    const int R = g.R;
    const size_t n = static_cast<size_t>(R) * g.pz;  // R whole planes (pitched)
    nck(nccl().GroupStart(), "ncclGroupStart");
    if (c->rank > 0) {
        nck(nccl().Send(row + R * g.pz, n, ncclFloat32, c->rank - 1, c->nc, s), "ncclSend");
        nck(nccl().Recv(row, n, ncclFloat32, c->rank - 1, c->nc, s), "ncclRecv");
    }
    if (c->rank < c->world - 1) {
        nck(nccl().Send(row + (g.Pz - 2 * R) * g.pz, n, ncclFloat32, c->rank + 1, c->nc, s),
            "ncclSend");
        nck(nccl().Recv(row + (g.Pz - R) * g.pz, n, ncclFloat32, c->rank + 1, c->nc, s),
            "ncclRecv");
    }
    nck(nccl().GroupEnd(), "ncclGroupEnd");
}

void slab_of(long pz_global, int R, int world, int rank, long* z_begin, long* z_end) {
    const long n = pz_global - 2L * R;
    *z_begin = R + n * rank / world;
    *z_end = R + n * (rank + 1) / world;
}

}  // namespace sfdb200
