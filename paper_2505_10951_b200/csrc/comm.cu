// comm.cu -- NCCL and host-callback transports for the multi-GPU exchanges (comm.cuh).
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "comm.cuh"
#include "common.cuh"

namespace sgc {
namespace {

// ---- the slice of the NCCL C ABI used here (nccl.h 2.x; the ABI is stable across 2.x) --------
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// libnccl.so.2 at run time: the copy already in the process (torch's) if there is one, else the
// loader's search path
const NcclApi* nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [h](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        if (api.GetUniqueId && api.CommInitRank && api.AllGather && api.Send && api.Recv &&
            api.GroupStart && api.GroupEnd && api.CommDestroy)
            api.h = h;
    });
    return api.h ? &api : nullptr;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != 0) {
        const NcclApi* a = nccl();
        fail(SGC_CUDA, std::string(what) + ": " + (a && a->GetErrorString ? a->GetErrorString(r) : "nccl error"));
    }
}

const NcclApi& nccl_or_fail() {
    const NcclApi* a = nccl();
    if (!a) fail(SGC_CUDA, "libnccl.so.2 not found (NCCL transport unavailable)");
    return *a;
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) nccl()->CommDestroy(comm);
    }
    void allgather(Ctx* c, const void* send, void* recv, size_t bytes) override {
        nccl_check(nccl()->AllGather(send, recv, bytes, kNcclUint8, comm, c->stream), "ncclAllGather");
    }
    void exchange(Ctx* c, const std::vector<P2P>& sends, const std::vector<P2P>& recvs) override {
        if (sends.empty() && recvs.empty()) return;
        const NcclApi* a = nccl();
        nccl_check(a->GroupStart(), "ncclGroupStart");
        for (const P2P& s : sends) nccl_check(a->Send(s.buf, s.bytes, kNcclUint8, s.peer, comm, c->stream), "ncclSend");
        for (const P2P& r : recvs) nccl_check(a->Recv(r.buf, r.bytes, kNcclUint8, r.peer, comm, c->stream), "ncclRecv");
        nccl_check(a->GroupEnd(), "ncclGroupEnd");
    }
    const char* kind() const override { return "nccl"; }
};

// host transport: device data staged through pinned host buffers around the callbacks
struct HostComm final : Comm {
    sgc_host_transport t{};
    void allgather(Ctx* c, const void* send, void* recv, size_t bytes) override {
        std::vector<uint8_t> hs(bytes), hr(bytes * world);
        SGC_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDefault, c->stream));
        SGC_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        if (t.allgather(t.user, hs.data(), hr.data(), bytes) != 0) fail(SGC_CUDA, "host transport: allgather failed");
        SGC_CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyDefault, c->stream));
        SGC_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    void exchange(Ctx* c, const std::vector<P2P>& sends, const std::vector<P2P>& recvs) override {
        std::vector<std::vector<uint8_t>> sb(sends.size()), rb(recvs.size());
        std::vector<const void*> sp;
        std::vector<void*> rp;
        std::vector<size_t> sn, rn;
        std::vector<int> speer, rpeer;
        for (size_t i = 0; i < sends.size(); ++i) {
            sb[i].resize(sends[i].bytes);
            SGC_CUDA_CHECK(cudaMemcpyAsync(sb[i].data(), sends[i].buf, sends[i].bytes, cudaMemcpyDefault, c->stream));
            sp.push_back(sb[i].data());
            sn.push_back(sends[i].bytes);
            speer.push_back(sends[i].peer);
        }
        SGC_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < recvs.size(); ++i) {
            rb[i].resize(recvs[i].bytes);
            rp.push_back(rb[i].data());
            rn.push_back(recvs[i].bytes);
            rpeer.push_back(recvs[i].peer);
        }
        if (t.exchange(t.user, static_cast<int>(sp.size()), sp.data(), sn.data(), speer.data(),
                       static_cast<int>(rp.size()), rp.data(), rn.data(), rpeer.data()) != 0)
            fail(SGC_CUDA, "host transport: exchange failed");
        for (size_t i = 0; i < recvs.size(); ++i)
            SGC_CUDA_CHECK(cudaMemcpyAsync(recvs[i].buf, rb[i].data(), rb[i].size(), cudaMemcpyDefault, c->stream));
        SGC_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    const char* kind() const override { return "host"; }
};

}  // namespace

bool nccl_available() { return nccl() != nullptr; }

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    nccl_check(nccl_or_fail().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

Comm* comm_nccl(Ctx* c, const uint8_t unique_id[128], int world, int rank) {
    const NcclApi& a = nccl_or_fail();
    ncclUniqueId id;
    std::memcpy(id.internal, unique_id, 128);
    auto* comm = new NcclComm();
    comm->rank = rank;
    comm->world = world;
    ncclResult_t r = a.CommInitRank(&comm->comm, world, id, rank);
    if (r != 0) {
        delete comm;
        nccl_check(r, "ncclCommInitRank");
    }
    (void)c;
    return comm;
}

Comm* comm_host(const sgc_host_transport* t, int world, int rank) {
    if (!t || !t->allgather || !t->exchange) fail(SGC_DOMAIN, "host transport needs allgather and exchange callbacks");
    auto* comm = new HostComm();
    comm->t = *t;
    comm->rank = rank;
    comm->world = world;
    return comm;
}

}  // namespace sgc
