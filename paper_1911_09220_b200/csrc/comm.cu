// Multi-GPU communication inside the library: an NCCL
// communicator per rank and the two collectives of a distributed CG
// iteration, enqueued on the context's stream -- so the distributed
// iteration is stream-ordered end to end and CUDA-graph capturable, and C++
// callers get multi-GPU through the C ABI alone.
//
//   halo update of p    ncclGroupStart; ncclSend / ncclRecv per peer;
//                       ncclGroupEnd (the owner's planes to the ghost copies)
//   dot products        ncclAllReduce(sum) of 1-2 doubles in place
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): a process that
// already loaded NCCL (e.g. torch's) shares that instance; a single-GPU
// process never needs it.
#include "common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

namespace tfem {
namespace {

struct NcclApi {
   ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
   ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
   ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
   ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
   ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                        cudaStream_t) = nullptr;
   ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
   ncclResult_t (*groupStart)() = nullptr;
   ncclResult_t (*groupEnd)() = nullptr;
   const char *(*getErrorString)(ncclResult_t) = nullptr;
   std::string error;
};

const NcclApi &api()
{
   static const NcclApi a = [] {
      NcclApi x;
      void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) {
         x.error = std::string("NCCL not found: ") + dlerror();
         return x;
      }
      auto sym = [&](auto &fn, const char *name) {
         fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
         if (!fn && x.error.empty()) x.error = std::string("NCCL symbol missing: ") + name;
      };
      sym(x.getUniqueId, "ncclGetUniqueId");
      sym(x.commInitRank, "ncclCommInitRank");
      sym(x.commDestroy, "ncclCommDestroy");
      sym(x.allReduce, "ncclAllReduce");
      sym(x.send, "ncclSend");
      sym(x.recv, "ncclRecv");
      sym(x.groupStart, "ncclGroupStart");
      sym(x.groupEnd, "ncclGroupEnd");
      sym(x.getErrorString, "ncclGetErrorString");
      return x;
   }();
   if (!a.error.empty()) throw Error(TFEM_CUDA_ERROR, a.error);
   return a;
}

void nccl_check(ncclResult_t r, const char *what)
{
   if (r != ncclSuccess)
      throw Error(TFEM_CUDA_ERROR, std::string(what) + ": " + api().getErrorString(r));
}

} // namespace

void nccl_unique_id(unsigned char *id)
{
   static_assert(sizeof(ncclUniqueId) == TFEM_NCCL_ID_BYTES, "ncclUniqueId size");
   ncclUniqueId u;
   nccl_check(api().getUniqueId(&u), "ncclGetUniqueId");
   std::memcpy(id, &u, sizeof(u));
}

tfem_nccl *nccl_create(tfem_ctx *ctx, int nranks, int rank, const unsigned char *id)
{
   if (nranks < 1 || rank < 0 || rank >= nranks) invalid("tfem_nccl_create: bad rank / size");
   ncclUniqueId u;
   std::memcpy(&u, id, sizeof(u));
   auto *c = new tfem_nccl;
   c->ctx = ctx;
   c->rank = rank;
   c->nranks = nranks;
   ncclComm_t comm = nullptr;
   const ncclResult_t r = api().commInitRank(&comm, nranks, u, rank);
   c->comm = comm;
   if (r != ncclSuccess) {
      delete c;
      nccl_check(r, "ncclCommInitRank");
   }
   return c;
}

void nccl_retain(tfem_nccl *c) { c->refs++; }

void nccl_destroy(tfem_nccl *c)
{
   if (--c->refs > 0) return;
   if (c->comm) api().commDestroy(static_cast<ncclComm_t>(c->comm));
   delete c;
}

// Sum k doubles in place over the ranks, on the context stream.
void nccl_allreduce(tfem_ctx *ctx, const tfem_nccl *c, double *d, int64_t k)
{
   nccl_check(api().allReduce(d, d, static_cast<size_t>(k), ncclFloat64, ncclSum,
                              static_cast<ncclComm_t>(c->comm),
                              ctx->stream),
              "ncclAllReduce");
}

// The halo update's transfers: every peer's send buffer out, its receive
// buffer in, one NCCL group (deadlock-free in any peer order).
void nccl_exchange(tfem_ctx *ctx, const tfem_operator *op, cudaStream_t s)
{
   (void)ctx;
   const NcclApi &a = api();
   nccl_check(a.groupStart(), "ncclGroupStart");
   for (int k = 0; k < op->n_peers; k++) {
      if (op->n_send[k] > 0)
         nccl_check(a.send(op->send_buf[k], static_cast<size_t>(op->n_send[k]), ncclFloat64,
                           op->peer_rank[k], static_cast<ncclComm_t>(op->nccl->comm), s),
                    "ncclSend");
      if (op->n_recv[k] > 0)
         nccl_check(a.recv(op->recv_buf[k], static_cast<size_t>(op->n_recv[k]), ncclFloat64,
                           op->peer_rank[k], static_cast<ncclComm_t>(op->nccl->comm), s),
                    "ncclRecv");
   }
   nccl_check(a.groupEnd(), "ncclGroupEnd");
}

} // namespace tfem
