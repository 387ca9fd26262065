// comm.cuh -- the two exchanges of the multi-GPU hot path, inside the library.
//
// Clusters shard across GPUs with no collective on the data path except:
//   * the all-gather of subgraph embeddings before clustering (every rank encodes a shard),
//   * the gather of per-query outputs to rank 0 (first token, logits, timings),
// plus, for clusters split across ranks at member level, a point-to-point
// copy of the sealed prefix K/V from the rank that prefilled it to the ranks serving the rest of
// its members (the reference's fork shares the sealed prefix by pointer, cache_engine.cpp:183).
//
// Two transports behind one interface:
//   * NCCL over NVLink / NVSwitch (libnccl.so.2 resolved at run time with dlopen, so the library
//     builds and loads without NCCL and shares the copy torch already loaded);
//   * a host transport: C callbacks over host buffers (e.g. torch.distributed gloo in the CPU
//     tests, or two in-process ranks in the C++ facade test).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

#include "sgc_b200.h"

namespace sgc {

struct Ctx;

struct P2P {
    void* buf;     // device memory (recv) / const device memory (send)
    size_t bytes;
    int peer;
};

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // recv[world * bytes] <- every rank's send[bytes], in rank order (device buffers)
    virtual void allgather(Ctx* c, const void* send, void* recv, size_t bytes) = 0;
    // one grouped exchange: all sends and receives of this rank posted together (no ordering
    // deadlock between ranks); returns when the stream has them queued (NCCL) or done (host)
    virtual void exchange(Ctx* c, const std::vector<P2P>& sends, const std::vector<P2P>& recvs) = 0;
    virtual const char* kind() const = 0;
};

Comm* comm_nccl(Ctx* c, const uint8_t unique_id[128], int world, int rank);
Comm* comm_host(const sgc_host_transport* t, int world, int rank);
void nccl_unique_id(uint8_t out[128]);
bool nccl_available();

}  // namespace sgc
