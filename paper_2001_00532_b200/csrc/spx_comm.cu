// Multi-GPU collectives of SURVEY.md §8(b)/(e): the final row gather of the
// row-sharded kernels (SpMV/SpMM/SDDMM) and the partial-result reduction of
// leaf-exact CSF shards (MTTKRP/TTV), as NCCL calls on caller streams.
//
// libnccl is opened lazily with dlopen (libnccl.so.2): libspx.so keeps no
// link-time NCCL dependency, still loads on a host without NCCL, and shares
// the copy torch has already loaded in the same process (dlopen returns the
// loaded library for a matching soname).  Communicators are opaque handles
// owned by the caller; the library never allocates device memory.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "spx_internal.h"

namespace spx {
namespace {

struct NcclId {
  char internal[128];  // NCCL_UNIQUE_ID_BYTES
};
typedef void* NcclComm;
typedef int (*GetUniqueId_t)(NcclId*);
typedef int (*CommInitRank_t)(NcclComm*, int, NcclId, int);
typedef int (*CommInitAll_t)(NcclComm*, int, const int*);
typedef int (*CommDestroy_t)(NcclComm);
typedef int (*CommCount_t)(NcclComm, int*);
typedef int (*CommUserRank_t)(NcclComm, int*);
typedef int (*AllGather_t)(const void*, void*, size_t, int, NcclComm, cudaStream_t);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*GroupStart_t)();
typedef int (*GroupEnd_t)();
typedef const char* (*GetErrorString_t)(int);

// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0;

struct Nccl {
  bool ok = false;
  std::string why;
  GetUniqueId_t get_id;
  CommInitRank_t init_rank;
  CommInitAll_t init_all;
  CommDestroy_t destroy;
  CommCount_t count;
  CommUserRank_t user_rank;
  AllGather_t all_gather;
  AllReduce_t all_reduce;
  GroupStart_t group_start;
  GroupEnd_t group_end;
  GetErrorString_t err_str;
};

std::mutex g_mu;
Nccl g_nccl;
bool g_tried = false;

const Nccl& nccl() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_tried) return g_nccl;
  g_tried = true;
  void* h = nullptr;
  for (const char* n : {"libnccl.so.2", "libnccl.so"})
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    g_nccl.why = "libnccl.so.2 not found";
    return g_nccl;
  }
#define SPX_SYM(field, name)                                                  \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));    \
  if (!g_nccl.field) {                                                        \
    g_nccl.why = std::string("missing symbol ") + name;                      \
    return g_nccl;                                                            \
  }
  SPX_SYM(get_id, "ncclGetUniqueId");
  SPX_SYM(init_rank, "ncclCommInitRank");
  SPX_SYM(init_all, "ncclCommInitAll");
  SPX_SYM(destroy, "ncclCommDestroy");
  SPX_SYM(count, "ncclCommCount");
  SPX_SYM(user_rank, "ncclCommUserRank");
  SPX_SYM(all_gather, "ncclAllGather");
  SPX_SYM(all_reduce, "ncclAllReduce");
  SPX_SYM(group_start, "ncclGroupStart");
  SPX_SYM(group_end, "ncclGroupEnd");
  SPX_SYM(err_str, "ncclGetErrorString");
#undef SPX_SYM
  g_nccl.ok = true;
  return g_nccl;
}

int check_nccl(const Nccl& n, int r, const char* what) {
  if (r == 0) return SPX_OK;
  return fail(SPX_E_CUDA, "%s: NCCL error %d (%s)", what, r, n.err_str ? n.err_str(r) : "?");
}

int nccl_type(int dtype, int* out) {
  switch (dtype) {
    case SPX_F64: *out = kNcclFloat64; return SPX_OK;
    case SPX_F32: *out = kNcclFloat32; return SPX_OK;
    case SPX_I32: *out = kNcclInt32; return SPX_OK;
    default: return fail(SPX_E_ARG, "collective: unknown dtype %d", dtype);
  }
}

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" {

int spx_comm_available(void) { return nccl().ok ? 1 : 0; }

int spx_comm_unique_id(void* id_out) {
  if (!id_out) return fail(SPX_E_ARG, "spx_comm_unique_id: null output");
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  NcclId id;
  if (int e = check_nccl(n, n.get_id(&id), "ncclGetUniqueId")) return e;
  std::memcpy(id_out, &id, sizeof(id));
  return SPX_OK;
}

int spx_comm_init(int nranks, int rank, const void* id, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(SPX_E_ARG, "spx_comm_init: bad arguments (nranks=%d rank=%d)", nranks, rank);
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  NcclId uid;
  std::memcpy(&uid, id, sizeof(uid));
  NcclComm c = nullptr;
  if (int e = check_nccl(n, n.init_rank(&c, nranks, uid, rank), "ncclCommInitRank")) return e;
  *comm_out = c;
  return SPX_OK;
}

int spx_comm_init_all(int ndev, const int* devs, void** comms_out) {
  if (ndev < 1 || !comms_out) return fail(SPX_E_ARG, "spx_comm_init_all: bad arguments");
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  return check_nccl(n, n.init_all(reinterpret_cast<NcclComm*>(comms_out), ndev, devs), "ncclCommInitAll");
}

int spx_comm_destroy(void* comm) {
  if (!comm) return SPX_OK;
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  return check_nccl(n, n.destroy(comm), "ncclCommDestroy");
}

int spx_comm_info(void* comm, int* nranks, int* rank) {
  const Nccl& n = nccl();
  if (!n.ok || !comm || !nranks || !rank) return fail(SPX_E_ARG, "spx_comm_info: bad arguments");
  if (int e = check_nccl(n, n.count(comm, nranks), "ncclCommCount")) return e;
  return check_nccl(n, n.user_rank(comm, rank), "ncclCommUserRank");
}

int spx_comm_group(int begin) {
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  return check_nccl(n, begin ? n.group_start() : n.group_end(), begin ? "ncclGroupStart" : "ncclGroupEnd");
}

// Row gather: every rank contributes `count` elements (its row shard padded
// to the largest shard) and receives nranks*count, rank-major.
int spx_gather(void* comm, const void* send, void* recv, size_t count, int dtype, void* stream) {
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  if (!comm || (count && (!send || !recv))) return fail(SPX_E_ARG, "spx_gather: null argument");
  int t = 0;
  if (int e = nccl_type(dtype, &t)) return e;
  return check_nccl(n, n.all_gather(send, recv, count, t, comm, static_cast<cudaStream_t>(stream)),
                    "ncclAllGather");
}

// Partial-result reduction (sum) of the dense outputs of leaf-exact shards;
// in place when send == recv.
int spx_reduce_rows(void* comm, const void* send, void* recv, size_t count, int dtype, void* stream) {
  const Nccl& n = nccl();
  if (!n.ok) return fail(SPX_E_UNSUPPORTED, "NCCL unavailable: %s", n.why.c_str());
  if (!comm || (count && (!send || !recv))) return fail(SPX_E_ARG, "spx_reduce_rows: null argument");
  int t = 0;
  if (int e = nccl_type(dtype, &t)) return e;
  return check_nccl(n, n.all_reduce(send, recv, count, t, kNcclSum, comm, static_cast<cudaStream_t>(stream)),
                    "ncclAllReduce");
}

}  // extern "C"
