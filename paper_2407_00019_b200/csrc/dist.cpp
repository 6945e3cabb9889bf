// dist.cpp -- multi-GPU row-block SpMV behind the C ABI (one process per GPU,
// NCCL over NVLink / NVSwitch).
//
// The reference's only split rule is partition_range (spmv.cpp:36-54): lane
// k of L gets a contiguous range of rows.  Across GPUs the ranges are
// entry-balanced (gen::partition_rows: rank k's first row is the first whose
// start reaches k*nnz/world), so a power-law matrix gets equal work per GPU,
// not equal rows.  Every transform is row-local (a shard converts on its own
// GPU with no communication); the only exchange is the iterate's x: after
// each SpMV every rank's block of x_{t+1} is broadcast to the others
// (grouped ncclBroadcast, in place: an all-gather with per-rank counts).
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is loaded at run time (below)

#include <cstring>
#include <mutex>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "generators.hpp"
#include "matrix.hpp"
#include "runtime.hpp"
#include "spmvtk/error.hpp"
#include "spmvtk/spmvtk.h"

struct spmvtk_dist {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  ~spmvtk_dist();
};

namespace spmvtk::dist {

namespace {
// NCCL is resolved at run time, not linked: a process that already holds an
// NCCL (PyTorch's, loaded first) must keep using that one -- two copies under
// one soname break whichever loads second -- and the library must load in
// processes that never touch multi-GPU.  Order: the NCCL already in the
// process, else libnccl.so.2 from the loader path.
struct Nccl {
  decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&::ncclCommInitRank) commInitRank = nullptr;
  decltype(&::ncclCommDestroy) commDestroy = nullptr;
  decltype(&::ncclAllGather) allGather = nullptr;
  decltype(&::ncclBroadcast) broadcast = nullptr;
  decltype(&::ncclGroupStart) groupStart = nullptr;
  decltype(&::ncclGroupEnd) groupEnd = nullptr;
  decltype(&::ncclGetErrorString) getErrorString = nullptr;
};

const Nccl& nccl() {
  static Nccl lib;
  static std::once_flag once;
  static std::string error;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      error = std::string("NCCL not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && error.empty()) error = std::string("NCCL symbol missing: ") + name;
    };
    sym(lib.getUniqueId, "ncclGetUniqueId");
    sym(lib.commInitRank, "ncclCommInitRank");
    sym(lib.commDestroy, "ncclCommDestroy");
    sym(lib.allGather, "ncclAllGather");
    sym(lib.broadcast, "ncclBroadcast");
    sym(lib.groupStart, "ncclGroupStart");
    sym(lib.groupEnd, "ncclGroupEnd");
    sym(lib.getErrorString, "ncclGetErrorString");
  });
  if (!error.empty()) throw Error(ErrorCode::Validation, error);
  return lib;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw Error(ErrorCode::Validation,
              std::string(what) + ": NCCL error " + nccl().getErrorString(r));
}
}  // namespace

spmvtk_dist* init(int rank, int world, const unsigned char* id) {
  if (world < 1 || rank < 0 || rank >= world)
    throw Error(ErrorCode::InvalidArgument, "rank must lie in [0, world)");
  static_assert(sizeof(ncclUniqueId) == SPMVTK_DIST_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  rt::init();
  auto d = std::make_unique<spmvtk_dist>();
  d->rank = rank;
  d->world = world;
  rt::check(cudaGetDevice(&d->device), "cudaGetDevice");
  nccl_check(nccl().commInitRank(&d->comm, world, uid, rank), "ncclCommInitRank");
  return d.release();
}

void destroy(spmvtk_dist* d) { delete d; }
void release(ncclComm_t c) {
  if (c) nccl().commDestroy(c);
}
int rank_of(const spmvtk_dist& d) { return d.rank; }
int world_of(const spmvtk_dist& d) { return d.world; }

void unique_id(unsigned char* out) {
  ncclUniqueId uid;
  nccl_check(nccl().getUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

// every rank's [row_offset, row_offset + rows) as begin[world + 1]
std::vector<std::int64_t> row_blocks(const spmvtk_dist& d, const dev::Matrix& shard) {
  rt::DevArray<std::int64_t> mine(2, "row blocks"), all(2 * static_cast<std::size_t>(d.world),
                                                         "row blocks");
  const std::int64_t h[2] = {shard.row_offset, shard.n};
  rt::copy_to_device(mine.get(), h, sizeof(h));
  nccl_check(nccl().allGather(mine.get(), all.get(), 2, ncclInt64, d.comm, rt::stream()),
             "row-block exchange");
  std::vector<std::int64_t> ha(2 * static_cast<std::size_t>(d.world));
  rt::copy_to_host(ha.data(), all.get(), ha.size() * sizeof(std::int64_t));
  std::vector<std::int64_t> begin(static_cast<std::size_t>(d.world) + 1);
  for (int r = 0; r < d.world; ++r) {
    begin[static_cast<std::size_t>(r)] = ha[2 * static_cast<std::size_t>(r)];
    if (r > 0 && ha[2 * static_cast<std::size_t>(r)] !=
                     ha[2 * static_cast<std::size_t>(r) - 2] + ha[2 * static_cast<std::size_t>(r) - 1])
      throw Error(ErrorCode::InvalidArgument, "shards do not tile the rows in rank order");
  }
  begin[static_cast<std::size_t>(d.world)] =
      ha[2 * static_cast<std::size_t>(d.world) - 2] + ha[2 * static_cast<std::size_t>(d.world) - 1];
  if (begin[0] != 0 || begin[static_cast<std::size_t>(d.world)] != shard.ncols)
    throw Error(ErrorCode::InvalidArgument, "shards do not cover the matrix rows");
  return begin;
}

// x_{t+1} = A x_t for `steps` steps; x (device, n = ncols doubles) holds x_0
// on entry and x_steps on exit on every rank.  Returns this rank's device
// seconds per step (the caller takes the max over ranks).
double iterate(const spmvtk_dist& d, const dev::Matrix& shard, spmvtk_kernel kernel, double* x,
               std::int64_t steps) {
  if (steps < 0) throw Error(ErrorCode::InvalidArgument, "steps must be >= 0");
  const std::int64_t n = shard.ncols;
  const std::vector<std::int64_t> begin = row_blocks(d, shard);
  rt::DevArray<double> other(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)), "x_{t+1}");
  cudaStream_t st = rt::stream();
  double* cur = x;
  double* nxt = other.get();
  auto exchange = [&](double* buf) {
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    for (int r = 0; r < d.world; ++r) {
      const std::int64_t b0 = begin[static_cast<std::size_t>(r)],
                         cnt = begin[static_cast<std::size_t>(r) + 1] - b0;
      if (cnt > 0)
        nccl_check(nccl().broadcast(buf + b0, buf + b0, static_cast<std::size_t>(cnt), ncclDouble, r,
                                 d.comm, st),
                   "x exchange");
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  };
  rt::EventTimer timer;
  timer.start();
  for (std::int64_t t = 0; t < steps; ++t) {
    // this rank's rows of x_{t+1}, written straight into its block
    if (shard.n > 0) dev::spmv_device(shard, kernel, cur, nxt + shard.row_offset);
    if (d.world > 1) exchange(nxt);
    std::swap(cur, nxt);
  }
  const double secs = timer.stop_seconds();
  if (cur != x)
    rt::check(cudaMemcpyAsync(x, cur, static_cast<std::size_t>(n) * sizeof(double),
                              cudaMemcpyDeviceToDevice, st),
              "iterate result");
  rt::sync();
  return steps > 0 ? secs / static_cast<double>(steps) : 0.0;
}

}  // namespace spmvtk::dist

spmvtk_dist::~spmvtk_dist() { spmvtk::dist::release(comm); }
