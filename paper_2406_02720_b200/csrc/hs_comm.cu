// hs_comm.cu -- the multi-GPU exchange step of the view-sharded training step
// (SURVEY.md 8(e)): every rank renders its views against a replica of the
// Gaussians, and the per-Gaussian gradients are summed over ranks.  The
// reference has no distributed path; its accumulation rule is GradientSet.add
// (rasterizer.py:100-105), a plain elementwise sum.
//
// hs_grad_allreduce sums one primitive range [begin, end) of every gradient
// field (and the touch counts) in ONE NCCL group -- ncclGroupStart, an
// ncclAllReduce per field slice, ncclGroupEnd -- so a bucket of K7's output is
// a single grouped launch on the caller's stream.  Issued on a side stream
// after each K7 bucket, the exchange of bucket b runs under the K7 of bucket
// b + 1 over NVLink/NVSwitch (NCCL selects NVLS when the node supports it).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): a process that already
// loaded NCCL (torch does) shares that copy; a host without NCCL still loads the
// library and gets HS_ERR_CUDA from these entry points only.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/halfsplat_b200.h"
#include "hs_common.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*comm_count)(const ncclComm_t, int*);
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*);
  ncclResult_t (*get_version)(int*);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t);
  ncclResult_t (*group_start)();
  ncclResult_t (*group_end)();
  bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

template <typename F>
bool bind(void* h, const char* name, F*& fn) {
  fn = reinterpret_cast<F*>(dlsym(h, name));
  return fn != nullptr;
}

const NcclApi* nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    NcclApi& a = g_nccl;
    a.ok = bind(h, "ncclGetUniqueId", a.get_unique_id) &&
           bind(h, "ncclCommInitRank", a.comm_init_rank) &&
           bind(h, "ncclCommDestroy", a.comm_destroy) && bind(h, "ncclCommCount", a.comm_count) &&
           bind(h, "ncclCommUserRank", a.comm_user_rank) &&
           bind(h, "ncclGetVersion", a.get_version) && bind(h, "ncclAllReduce", a.all_reduce) &&
           bind(h, "ncclGroupStart", a.group_start) && bind(h, "ncclGroupEnd", a.group_end);
  });
  return g_nccl.ok ? &g_nccl : nullptr;
}

}  // namespace

static_assert(sizeof(ncclUniqueId) == HS_COMM_ID_BYTES, "ncclUniqueId size");

extern "C" int hs_comm_unique_id(void* id) {
  const NcclApi* a = nccl();
  if (!a) return HS_ERR_CUDA;
  if (!id) return HS_ERR_INVALID_ARG;
  ncclUniqueId u;
  if (a->get_unique_id(&u) != ncclSuccess) return HS_ERR_CUDA;
  memcpy(id, &u, sizeof(u));
  return HS_OK;
}

extern "C" int hs_comm_init(void** comm, int32_t world, int32_t rank, const void* id) {
  const NcclApi* a = nccl();
  if (!a) return HS_ERR_CUDA;
  if (!comm || !id || world <= 0 || rank < 0 || rank >= world) return HS_ERR_INVALID_ARG;
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  if (a->comm_init_rank(&c, world, u, rank) != ncclSuccess) return HS_ERR_CUDA;
  *comm = c;
  return HS_OK;
}

extern "C" int hs_comm_destroy(void* comm) {
  const NcclApi* a = nccl();
  if (!a) return HS_ERR_CUDA;
  if (!comm) return HS_OK;
  return a->comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? HS_OK : HS_ERR_CUDA;
}

extern "C" int hs_comm_info(void* comm, int32_t* world, int32_t* rank, int32_t* nccl_version) {
  const NcclApi* a = nccl();
  if (!a) return HS_ERR_CUDA;
  int v = 0;
  if (nccl_version && a->get_version(&v) == ncclSuccess) *nccl_version = v;
  if (!comm) return HS_OK;
  int n = 0, r = 0;
  if (a->comm_count(static_cast<ncclComm_t>(comm), &n) != ncclSuccess ||
      a->comm_user_rank(static_cast<ncclComm_t>(comm), &r) != ncclSuccess)
    return HS_ERR_CUDA;
  if (world) *world = n;
  if (rank) *rank = r;
  return HS_OK;
}

extern "C" int hs_grad_allreduce(void* comm, const hs_grads* g, int64_t n, int32_t sh_degree,
                                 int32_t dtype, int64_t begin, int64_t end, int32_t with_touch,
                                 void* stream) {
  const NcclApi* a = nccl();
  if (!a) return HS_ERR_CUDA;
  if (!comm || !g || n < 0 || sh_degree < 0 || sh_degree > 3) return HS_ERR_INVALID_ARG;
  if (dtype != HS_DTYPE_F32 && dtype != HS_DTYPE_F64) return HS_ERR_INVALID_ARG;
  if (begin < 0 || end > n || begin > end) return HS_ERR_INVALID_ARG;
  const int64_t k = (int64_t)(sh_degree + 1) * (sh_degree + 1);
  const size_t es = dtype == HS_DTYPE_F32 ? 4 : 8;
  const ncclDataType_t t = dtype == HS_DTYPE_F32 ? ncclFloat32 : ncclFloat64;
  const int64_t cnt = end - begin;
  struct Field {
    void* p;
    int64_t width;
  } fields[] = {{g->d_mu, 3},
                {g->d_log_scale, 3},
                {g->d_rotation, 4},
                {g->d_sh, 3 * k},
                {g->d_normal, 3},
                {g->d_raw_opacity_a, 1},
                {g->d_raw_opacity_b, 1},
                {g->pos_grad_norm, 1}};
  for (const Field& f : fields)
    if (!f.p) return HS_ERR_INVALID_ARG;
  if (with_touch && !g->touch_count) return HS_ERR_INVALID_ARG;
  if (cnt == 0) return HS_OK;
  const ncclComm_t c = static_cast<ncclComm_t>(comm);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (a->group_start() != ncclSuccess) return HS_ERR_CUDA;
  ncclResult_t r = ncclSuccess;
  for (const Field& f : fields) {
    char* p = static_cast<char*>(f.p) + (size_t)(begin * f.width) * es;
    if (r == ncclSuccess) r = a->all_reduce(p, p, (size_t)(cnt * f.width), t, ncclSum, c, s);
  }
  if (with_touch && r == ncclSuccess)
    r = a->all_reduce(g->touch_count + begin, g->touch_count + begin, (size_t)cnt, ncclInt32,
                      ncclSum, c, s);
  const ncclResult_t e = a->group_end();
  return (r == ncclSuccess && e == ncclSuccess) ? HS_OK : HS_ERR_CUDA;
}
