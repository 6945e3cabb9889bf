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
#include <array>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "generators.hpp"
#include "matrix.hpp"
#include "runtime.hpp"
#include "spmvtk/error.hpp"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

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

// ---- the exchange folded into the SpMV (push over peer memory) -------------
// Every rank's two x buffers and its step flags are cudaMalloc memory shared
// through CUDA IPC (handles exchanged with one NCCL all-gather).  Step t: the
// pushed SpMV (spmvtk_k_spmv_*_push) first waits in its prologue until every
// source has flagged step t (its rows of x_t are in my buffer t%2, and it
// has finished reading the buffer I am about to overwrite), then stores each
// result row straight into buffer (t+1)%2 of every rank that reads it (the
// per-row mask, from the gathered column sets; all ranks without it), and
// its last CTA raises flag t+1 on every rank.  One launch per step, no
// collective; NVLink carries the stores while the SpMV computes.
struct Push {
  const spmvtk_dist* d = nullptr;
  const dev::Matrix* shard = nullptr;
  spmvtk_kernel kernel = SPMVTK_KERNEL_CRS;
  std::int64_t n = 0;
  void* own[3] = {nullptr, nullptr, nullptr};   // x0, x1, flags
  std::vector<void*> opened;                     // peers' mapped buffers
  std::vector<std::array<void*, 3>> peer;        // per rank: x0, x1, flags
  rt::DevArray<std::uint8_t> mask;
  rt::DevArray<std::uint32_t> status, counter;
  std::uint64_t timeout_ns = 10'000'000'000ull;
  ~Push();
};

namespace {
// a barrier that also agrees on a flag: true on every rank iff `ok` on all
// (so a local failure turns into the same error on every rank instead of
// leaving the others inside a collective)
bool all_ok(const spmvtk_dist& d, bool ok) {
  rt::DevArray<int> one(1, "barrier");
  cudaStream_t st = rt::stream();
  rt::check(cudaMemsetAsync(one.get(), ok ? 1 : 0, sizeof(int), st), "barrier");
  rt::DevArray<int> all(static_cast<std::size_t>(d.world), "barrier");
  nccl_check(nccl().allGather(one.get(), all.get(), 1, ncclInt32, d.comm, st), "barrier");
  std::vector<int> h(static_cast<std::size_t>(d.world));
  rt::copy_to_host(h.data(), all.get(), h.size() * sizeof(int));
  for (int v : h)
    if (v == 0) return false;
  return true;
}
void barrier(const spmvtk_dist& d) { (void)all_ok(d, true); }
}  // namespace

Push* push_create(const spmvtk_dist& d, const dev::Matrix& shard, spmvtk_kernel kernel,
                  bool sparse) {
  if (d.world > SPMVTK_MAX_PEERS)
    throw Error(ErrorCode::InvalidArgument, "the push exchange supports up to 8 ranks");
  if (shard.format != SPMVTK_FORMAT_CRS && shard.format != SPMVTK_FORMAT_ELL)
    throw Error(ErrorCode::InvalidArgument, "the push exchange takes a CRS or band-major ELL shard");
  (void)row_blocks(d, shard);  // the shards must tile the rows in rank order
  auto p = std::make_unique<Push>();
  p->d = &d;
  p->shard = &shard;
  p->kernel = kernel;
  p->n = shard.ncols;
  cudaStream_t st = rt::stream();
  // own buffers and their IPC handles; an error on one rank must not leave
  // the others in the collective: the handles are gathered either way and a
  // zero handle marks a failed rank
  unsigned char mine[3 * SPMVTK_IPC_HANDLE_BYTES] = {};
  bool ok = true;
  const std::size_t sizes[3] = {static_cast<std::size_t>(p->n) * 8,
                                static_cast<std::size_t>(p->n) * 8,
                                static_cast<std::size_t>(d.world) * 8};
  for (int b = 0; b < 3 && ok; ++b) {
    if (cudaMalloc(&p->own[b], std::max<std::size_t>(sizes[b], 8)) != cudaSuccess ||
        cudaMemset(p->own[b], 0, std::max<std::size_t>(sizes[b], 8)) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p->own[b]) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    std::memcpy(mine + b * SPMVTK_IPC_HANDLE_BYTES, &h, sizeof(h));
  }
  if (!ok) std::memset(mine, 0, sizeof(mine));
  rt::DevArray<unsigned char> dmine(sizeof(mine), "IPC handles"),
      dall(sizeof(mine) * static_cast<std::size_t>(d.world), "IPC handles");
  rt::copy_to_device(dmine.get(), mine, sizeof(mine));
  nccl_check(nccl().allGather(dmine.get(), dall.get(), sizeof(mine), ncclChar, d.comm, st),
             "IPC handle exchange");
  std::vector<unsigned char> all(sizeof(mine) * static_cast<std::size_t>(d.world));
  rt::copy_to_host(all.data(), dall.get(), all.size());
  auto zero = [](const unsigned char* h) {
    for (std::size_t i = 0; i < 3 * SPMVTK_IPC_HANDLE_BYTES; ++i)
      if (h[i]) return false;
    return true;
  };
  for (int w = 0; w < d.world; ++w)
    if (zero(all.data() + sizeof(mine) * static_cast<std::size_t>(w)))
      throw Error(ErrorCode::Validation, "push exchange: rank " + std::to_string(w) +
                                             " could not share its buffers");
  p->peer.resize(static_cast<std::size_t>(d.world));
  std::string open_error;
  for (int w = 0; w < d.world && open_error.empty(); ++w) {
    for (int b = 0; b < 3; ++b) {
      if (w == d.rank) {
        p->peer[static_cast<std::size_t>(w)][static_cast<std::size_t>(b)] = p->own[b];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, all.data() + sizeof(mine) * static_cast<std::size_t>(w) +
                          static_cast<std::size_t>(b) * SPMVTK_IPC_HANDLE_BYTES,
                  sizeof(h));
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        cudaGetLastError();
        open_error = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
        break;
      }
      p->opened.push_back(ptr);
      p->peer[static_cast<std::size_t>(w)][static_cast<std::size_t>(b)] = ptr;
    }
  }
  if (!all_ok(d, open_error.empty()))
    throw Error(ErrorCode::Validation,
                "push exchange: a rank could not map its peers' buffers" +
                    (open_error.empty() ? std::string() : " (here: " + open_error + ")"));
  if (sparse && d.world > 1) {  // which ranks read each of my rows
    rt::DevArray<std::uint8_t> need(static_cast<std::size_t>(std::max<std::int64_t>(p->n, 1)),
                                    "push mask");
    rt::check(cudaMemsetAsync(need.get(), 0, need.bytes(), st), "push mask");
    const std::int64_t cols = shard.format == SPMVTK_FORMAT_ELL
                                  ? static_cast<std::int64_t>(shard.col.size())
                                  : shard.nnz;
    rt::check_launch(spmvtk_k_mark_columns(shard.col.get(), cols, need.get(), st), "push mask");
    rt::DevArray<std::uint8_t> need_all(need.size() * static_cast<std::size_t>(d.world),
                                        "push mask");
    nccl_check(nccl().allGather(need.get(), need_all.get(), need.size(), ncclUint8, d.comm, st),
               "push mask exchange");
    p->mask.reset(static_cast<std::size_t>(std::max<std::int64_t>(shard.n, 1)), "push mask");
    rt::check_launch(spmvtk_k_push_mask(need_all.get(), d.world, static_cast<std::int64_t>(need.size()),
                                        shard.row_offset, shard.n, d.rank, p->mask.get(), st),
                     "push mask");
  }
  p->status.reset(1, "push status");
  p->counter.reset(1, "push counter");
  rt::check(cudaMemsetAsync(p->status.get(), 0, 4, st), "push status");
  rt::check(cudaMemsetAsync(p->counter.get(), 0, 4, st), "push counter");
  barrier(d);
  return p.release();
}

Push::~Push() {
  if (d) {
    try {
      barrier(*d);  // nobody pushes into or reads my buffers any more
    } catch (...) {
    }
  }
  for (void* q : opened) cudaIpcCloseMemHandle(q);
  for (void* q : own)
    if (q) cudaFree(q);
}

void push_free(Push* p) { delete p; }

double push_iterate(Push& p, double* x, std::int64_t steps) {
  if (steps < 0) throw Error(ErrorCode::InvalidArgument, "steps must be >= 0");
  const spmvtk_dist& d = *p.d;
  const dev::Matrix& shard = *p.shard;
  const std::vector<std::int64_t> begin = row_blocks(d, shard);
  cudaStream_t st = rt::stream();
  const std::size_t xb = static_cast<std::size_t>(p.n) * 8;
  // a fresh run: flags back to 0 everywhere before anyone pushes
  rt::check(cudaMemsetAsync(p.own[2], 0, static_cast<std::size_t>(d.world) * 8, st), "push reset");
  rt::check(cudaMemsetAsync(p.status.get(), 0, 4, st), "push reset");
  rt::check(cudaMemcpyAsync(p.own[0], x, xb, cudaMemcpyDeviceToDevice, st), "push x0");
  barrier(d);
  spmvtk_push push[2];
  for (int b = 0; b < 2; ++b) {
    std::memset(&push[b], 0, sizeof(push[b]));
    for (int w = 0; w < d.world; ++w)
      push[b].dst[w] = static_cast<double*>(p.peer[static_cast<std::size_t>(w)][static_cast<std::size_t>(b)]) +
                       shard.row_offset;
    push[b].mask = p.mask.size() ? p.mask.get() : nullptr;
    push[b].ndst = d.world;
    push[b].local = d.rank;
  }
  spmvtk_push_sync sync;
  std::memset(&sync, 0, sizeof(sync));
  sync.wait_flags = static_cast<const std::uint64_t*>(p.own[2]);
  sync.nwait = d.world;
  sync.timeout_ns = p.timeout_ns;
  sync.status = p.status.get();
  for (int w = 0; w < d.world; ++w)
    sync.signal.ptr[w] = static_cast<std::uint64_t*>(p.peer[static_cast<std::size_t>(w)][2]) + d.rank;
  sync.signal.n = d.world;
  sync.counter = p.counter.get();
  rt::EventTimer timer;
  timer.start();
  for (std::int64_t t = 0; t < steps; ++t) {
    sync.wait_value = static_cast<std::uint64_t>(t);
    sync.signal_value = static_cast<std::uint64_t>(t + 1);
    dev::spmv_device_push(shard, p.kernel, static_cast<const double*>(p.own[t % 2]),
                          push[(t + 1) % 2], &sync);
  }
  const double secs = timer.stop_seconds();
  // every source has finished pushing into my buffers
  rt::check_launch(spmvtk_k_flags_wait(static_cast<const std::uint64_t*>(p.own[2]), d.world,
                                       static_cast<std::uint64_t>(steps), p.timeout_ns,
                                       p.status.get(), st),
                   "push drain");
  std::uint32_t status = 0;
  rt::copy_to_host(&status, p.status.get(), 4);
  if (!all_ok(d, status == 0))  // agreed, so no rank is left in the broadcasts below
    throw Error(ErrorCode::Validation, "push exchange: a step flag wait timed out");
  // x_steps: own rows from my buffer, the other blocks from their owners
  // (with the sparse mask a buffer only holds the rows this rank reads)
  rt::check(cudaMemcpyAsync(x, p.own[steps % 2], xb, cudaMemcpyDeviceToDevice, st), "push result");
  if (d.world > 1) {
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    for (int r = 0; r < d.world; ++r) {
      const std::int64_t b0 = begin[static_cast<std::size_t>(r)],
                         cnt = begin[static_cast<std::size_t>(r) + 1] - b0;
      if (cnt > 0)
        nccl_check(nccl().broadcast(x + b0, x + b0, static_cast<std::size_t>(cnt), ncclDouble, r,
                                    d.comm, st),
                   "push result exchange");
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  }
  rt::sync();
  barrier(d);  // no rank starts the next run while a peer still reads
  return steps > 0 ? secs / static_cast<double>(steps) : 0.0;
}

}  // namespace spmvtk::dist

spmvtk_dist::~spmvtk_dist() { spmvtk::dist::release(comm); }
