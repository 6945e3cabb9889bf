// capi.cpp -- the C ABI (include/spmvtk/spmvtk.h).
//
// Error firewall as in /root/reference/proj/src/capi.cpp:33-62: every entry
// point catches, maps ErrorCode -> status (InvalidArgument -> USAGE,
// MemoryLimit -> MEMORY_LIMIT, the rest -> DATA), stores what() in a
// thread-local string and clears it on success.  No exception crosses the
// ABI.  Handles own device memory (matrix.hpp).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "autotune.hpp"
#include "generators.hpp"
#include "matrix.hpp"
#include "mmio.hpp"
#include "runtime.hpp"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk;

struct spmvtk_profile {
  at::Profile p;
};

namespace {

thread_local std::string t_error;

spmvtk_status to_status(ErrorCode c) {
  switch (c) {
    case ErrorCode::InvalidArgument: return SPMVTK_ERR_USAGE;
    case ErrorCode::MemoryLimit: return SPMVTK_ERR_MEMORY_LIMIT;
    default: return SPMVTK_ERR_DATA;
  }
}

template <typename F>
spmvtk_status guarded(F&& f) {
  try {
    f();
    t_error.clear();
    return SPMVTK_OK;
  } catch (const Error& e) {
    t_error = e.what();
    return to_status(e.code());
  } catch (const std::bad_alloc&) {
    t_error = "host allocation failed";
    return SPMVTK_ERR_MEMORY_LIMIT;
  } catch (const std::exception& e) {
    t_error = e.what();
    return SPMVTK_ERR_DATA;
  }
}

void need(const void* p, const char* msg = "null argument") {
  if (!p) throw Error(ErrorCode::InvalidArgument, msg);
}

const dev::Matrix& crs_of(const spmvtk_matrix* m) {
  if (!m) throw Error(ErrorCode::InvalidArgument, "null matrix handle");
  if (m->format != SPMVTK_FORMAT_CRS)
    throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
  return *m;
}

dev::Matrix* upload(const gen::HostCrs& h) {
  const std::int64_t ncols = h.ncols < 0 ? h.n : h.ncols;
  if (h.wide())
    return dev::crs_block_from_arrays(h.n, ncols, h.row_offset, h.nnz(), h.row_ptr.data(),
                                      h.col_idx.data(), h.values.data(), 8, h.base, false);
  return dev::crs_block_from_arrays(h.n, ncols, h.row_offset, h.nnz(), h.row_ptr32.data(),
                                    h.col32.data(), h.values.data(), 4, h.base, false);
}

thread_local double t_scratch = 0.0;

bool pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[8] = {};
  SideStream() {
    rt::check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "side stream");
    for (auto& e : ev) rt::check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
};

double pipelined_spmv(const dev::Matrix& m, spmvtk_kernel kernel, const double* dx, double* dy,
                      double* y_host) {
  thread_local SideStream side;
  constexpr int kChunks = 4;
  const std::int64_t n = m.n;
  std::int64_t step = (n + kChunks - 1) / kChunks;
  step = (step + 63) / 64 * 64;
  cudaStream_t st = rt::stream();
  rt::EventTimer timer;
  timer.start();
  int k = 0;
  for (std::int64_t r0 = 0; r0 < n; r0 += step, ++k) {
    const std::int64_t r1 = std::min(n, r0 + step);
    dev::spmv_device_rows(m, kernel, dx, dy, r0, r1);
    rt::check(cudaEventRecord(side.ev[k], st), "event");
    rt::check(cudaStreamWaitEvent(side.s, side.ev[k], 0), "event wait");
    rt::check(cudaMemcpyAsync(y_host + r0, dy + r0, static_cast<std::size_t>(r1 - r0) * 8,
                              cudaMemcpyDeviceToHost, side.s),
              "D2H copy");
  }
  const double secs = timer.stop_seconds();
  rt::check(cudaStreamSynchronize(side.s), "side stream synchronize");
  return secs;
}

bool valid_format(int f) { return f >= SPMVTK_FORMAT_CRS && f <= SPMVTK_FORMAT_ELL_ROWMAJOR; }
bool valid_kernel(int k) { return k >= SPMVTK_KERNEL_CRS && k <= SPMVTK_KERNEL_ELL_ROWMAJOR; }

// 1-based triplets of any handle (for the Matrix Market writer)
void triplets(const dev::Matrix& m, std::vector<std::int64_t>& r, std::vector<std::int64_t>& c,
              std::vector<double>& v) {
  auto get_idx = [&](spmvtk_array a) {
    std::int64_t len = dev::copy_array(m, a, nullptr, 0, 8, 1);
    std::vector<std::int64_t> out(static_cast<std::size_t>(len));
    dev::copy_array(m, a, out.data(), len, 8, 1);
    return out;
  };
  std::int64_t vl = dev::copy_array(m, SPMVTK_ARRAY_VALUES, nullptr, 0, 8, 1);
  std::vector<double> vals(static_cast<std::size_t>(vl));
  dev::copy_array(m, SPMVTK_ARRAY_VALUES, vals.data(), vl, 8, 1);
  switch (m.format) {
    case SPMVTK_FORMAT_CRS:
    case SPMVTK_FORMAT_CCS: {
      auto ptr = get_idx(SPMVTK_ARRAY_POINTER);
      auto idx = get_idx(m.format == SPMVTK_FORMAT_CRS ? SPMVTK_ARRAY_COL_IDX : SPMVTK_ARRAY_ROW_IDX);
      std::vector<std::int64_t> seg(idx.size());
      for (std::int64_t s = 1; s <= m.n; ++s)
        for (std::int64_t p = ptr[s - 1]; p < ptr[s]; ++p) seg[static_cast<std::size_t>(p - 1)] = s;
      if (m.format == SPMVTK_FORMAT_CRS) {
        r = std::move(seg);
        c = std::move(idx);
      } else {
        r = std::move(idx);
        c = std::move(seg);
      }
      v = std::move(vals);
      return;
    }
    case SPMVTK_FORMAT_COO_ROW:
    case SPMVTK_FORMAT_COO_COL:
      r = get_idx(SPMVTK_ARRAY_ROW_IDX);
      c = get_idx(SPMVTK_ARRAY_COL_IDX);
      v = std::move(vals);
      return;
    case SPMVTK_FORMAT_ELL:
    case SPMVTK_FORMAT_ELL_ROWMAJOR: {
      // drop exactly the padding slots using row_entry_count (convert.cpp:166-183)
      auto col = get_idx(SPMVTK_ARRAY_COL_IDX);
      std::int64_t cl = dev::copy_array(m, SPMVTK_ARRAY_ROW_ENTRY_COUNT, nullptr, 0, 8, 0);
      std::vector<std::int64_t> cnt(static_cast<std::size_t>(cl));
      dev::copy_array(m, SPMVTK_ARRAY_ROW_ENTRY_COUNT, cnt.data(), cl, 8, 0);
      const std::int64_t nz = m.band_count;
      for (std::int64_t i = 0; i < m.n; ++i)
        for (std::int64_t k = 0; k < cnt[static_cast<std::size_t>(i)]; ++k) {
          std::size_t s = m.format == SPMVTK_FORMAT_ELL ? static_cast<std::size_t>(k * m.n + i)
                                                        : static_cast<std::size_t>(i * nz + k);
          r.push_back(i + 1);
          c.push_back(col[s]);
          v.push_back(vals[s]);
        }
      return;
    }
  }
}

}  // namespace

extern "C" {

const char* spmvtk_last_error(void) { return t_error.c_str(); }

void spmvtk_matrix_free(spmvtk_matrix* m) {
  if (!m) return;
  // stream-ordered: the buffers go back to the pool once the work already
  // queued on the calling thread's stream has finished with them (no device
  // synchronisation).  Work the caller queued on OTHER streams must be
  // complete first, as with any freed buffer.
  delete m;
}

void spmvtk_profile_free(spmvtk_profile* p) { delete p; }

spmvtk_status spmvtk_read_matrix_market(const char* path, spmvtk_matrix** out) {
  return guarded([&] {
    need(path);
    need(out);
    *out = upload(mm::read(path));
  });
}

spmvtk_status spmvtk_write_matrix_market(const spmvtk_matrix* m, const char* path) {
  return guarded([&] {
    need(m);
    need(path);
    std::vector<std::int64_t> r, c;
    std::vector<double> v;
    if (m->format == SPMVTK_FORMAT_CRS) {
      triplets(*m, r, c, v);
    } else {
      // non-CRS handles are written through their canonical CRS, rebuilt on
      // the device (duplicates refused there, as coo_to_crs does)
      std::unique_ptr<dev::Matrix> crs(dev::to_crs(*m));
      triplets(*crs, r, c, v);
    }
    mm::write(m->n, std::move(r), std::move(c), std::move(v), false, path);
  });
}

spmvtk_status spmvtk_gen_banded(int64_t n, int64_t half_width, spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = upload(gen::banded(n, half_width));
  });
}

spmvtk_status spmvtk_gen_skewed(int64_t n, int64_t base_deg, int64_t heavy_rows,
                                int64_t heavy_deg, uint64_t seed, spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = upload(gen::skewed(n, base_deg, heavy_rows, heavy_deg, seed));
  });
}

spmvtk_status spmvtk_gen_cv_target(int64_t n, double mean_deg, double target_dmat,
                                   uint64_t seed, spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = upload(gen::cv_target(n, mean_deg, target_dmat, seed));
  });
}

spmvtk_format spmvtk_matrix_get_format(const spmvtk_matrix* m) {
  return m ? m->format : SPMVTK_FORMAT_CRS;
}

spmvtk_status spmvtk_matrix_get_info(const spmvtk_matrix* m, spmvtk_matrix_info* out) {
  return guarded([&] {
    need(out, "null output");
    const dev::Matrix& a = crs_of(m);
    out->n = a.n;
    out->nnz = a.nnz;
    rt::Moments mo = dev::crs_moments(a);
    out->max_row_entries = static_cast<int64_t>(mo.max);
    out->ell_bytes = static_cast<uint64_t>(a.n) * mo.max * 16ull;
    rt::RowStatsD s = rt::stats_from_moments(mo, a.n);
    out->mu = s.mu;
    out->sigma = s.sigma;
    out->d_mat = s.d_mat;
  });
}

spmvtk_status spmvtk_matrix_convert(const spmvtk_matrix* m, spmvtk_format to,
                                    uint64_t max_bytes, spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    const dev::Matrix& a = crs_of(m);
    if (!valid_format(to)) throw Error(ErrorCode::InvalidArgument, "unknown target format");
    *out = dev::convert(a, to, max_bytes);
  });
}

spmvtk_status spmvtk_matrix_convert_timed(const spmvtk_matrix* m, spmvtk_format to,
                                          uint64_t max_bytes, spmvtk_matrix** out,
                                          double* seconds) {
  return guarded([&] {
    need(out, "null output");
    need(seconds, "null output");
    const dev::Matrix& a = crs_of(m);
    if (!valid_format(to)) throw Error(ErrorCode::InvalidArgument, "unknown target format");
    auto [conv, secs] = at::measure_transformation(a, to, max_bytes);
    *out = conv;
    *seconds = secs;
  });
}

spmvtk_status spmvtk_spmv(const spmvtk_matrix* m, spmvtk_kernel kernel, const double* x,
                          int64_t len, int lanes, double* y, double* elapsed_seconds) {
  return guarded([&] {
    if (!m || !x || !y) throw Error(ErrorCode::InvalidArgument, "null argument");
    if (!valid_kernel(kernel)) throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
    if (kernel != SPMVTK_KERNEL_CRS && lanes < 1)
      throw Error(ErrorCode::InvalidArgument, "lane count must be at least 1");
    if (len != m->ncols)
      throw Error(ErrorCode::InvalidArgument, "vector length " + std::to_string(len) +
                                                  " does not match matrix dimension " +
                                                  std::to_string(m->ncols));
    rt::init();
    const std::size_t n = static_cast<std::size_t>(m->n);
    const std::size_t nc = static_cast<std::size_t>(m->ncols);
    rt::DevArray<double> dx(std::max<std::size_t>(nc, 1), "x"), dy(std::max<std::size_t>(n, 1), "y");
    rt::copy_to_device(dx.get(), x, nc * sizeof(double));
    if (n >= 16384 && dev::spmv_row_splittable(*m, kernel) && pinned(y)) {
      // pipelined: the D2H copy of each finished row block overlaps the
      // SpMV of the next (x must be complete before any row: gathers are
      // arbitrary), on a side stream ordered by events
      *(elapsed_seconds ? elapsed_seconds : &t_scratch) =
          pipelined_spmv(*m, kernel, dx.get(), dy.get(), y);
      return;
    }
    rt::EventTimer timer;
    timer.start();
    dev::spmv_device(*m, kernel, dx.get(), dy.get());
    double secs = timer.stop_seconds();
    rt::copy_to_host(y, dy.get(), n * sizeof(double));
    if (elapsed_seconds) *elapsed_seconds = secs;
  });
}

// ---- streaming host SpMV (spmvtk_pipeline_*) -------------------------------
struct spmvtk_pipeline {
  static constexpr int kMaxSplit = 4;
  static constexpr int kMaxSlots = 4;
  const dev::Matrix* m = nullptr;
  int slots = 3;  // device staging slots (products in flight): 3 measured 10-12 % faster
                  // than 2 and 4 at n = 2^20 (profiles/r01_pipeline_slots.txt),
                  // within 3 % of the PCIe duplex copy time; SPMVTK_PIPE_SLOTS overrides
  spmvtk_kernel kernel = SPMVTK_KERNEL_CRS;
  int split = 2;  // copies per direction cut into `split` parts on their own streams
                  // (2 measured 6 % faster than 1 and 4 at n = 2^20,
                  // profiles/r01_pipeline_split.txt; SPMVTK_PIPE_SPLIT overrides)
  cudaStream_t h2d[kMaxSplit] = {}, d2h[kMaxSplit] = {};
  cudaStream_t comp = nullptr;
  double* x[kMaxSlots] = {};
  double* y[kMaxSlots] = {};
  cudaEvent_t h2d_done[kMaxSlots][kMaxSplit] = {}, comp_done[kMaxSlots] = {},
              d2h_done[kMaxSlots][kMaxSplit] = {};
  std::uint64_t count = 0;
  ~spmvtk_pipeline() {
    if (comp) cudaStreamSynchronize(comp);
    for (int k = 0; k < kMaxSplit; ++k) {
      if (d2h[k]) cudaStreamSynchronize(d2h[k]);
      if (h2d[k]) cudaStreamSynchronize(h2d[k]);
    }
    for (int b = 0; b < kMaxSlots; ++b) {
      if (x[b]) cudaFree(x[b]);
      if (y[b]) cudaFree(y[b]);
      if (comp_done[b]) cudaEventDestroy(comp_done[b]);
      for (int k = 0; k < kMaxSplit; ++k) {
        if (h2d_done[b][k]) cudaEventDestroy(h2d_done[b][k]);
        if (d2h_done[b][k]) cudaEventDestroy(d2h_done[b][k]);
      }
    }
    for (int k = 0; k < kMaxSplit; ++k) {
      if (h2d[k]) cudaStreamDestroy(h2d[k]);
      if (d2h[k]) cudaStreamDestroy(d2h[k]);
    }
    if (comp) cudaStreamDestroy(comp);
  }
};

spmvtk_status spmvtk_pipeline_create(const spmvtk_matrix* m, spmvtk_kernel kernel,
                                     spmvtk_pipeline** out) {
  return guarded([&] {
    if (!m || !out) throw Error(ErrorCode::InvalidArgument, "null argument");
    if (!valid_kernel(kernel)) throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
    rt::init();
    auto p = std::make_unique<spmvtk_pipeline>();
    p->m = m;
    p->kernel = kernel;
    if (const char* e = std::getenv("SPMVTK_PIPE_SPLIT"))
      p->split = std::max(1, std::min(spmvtk_pipeline::kMaxSplit, std::atoi(e)));
    if (const char* e = std::getenv("SPMVTK_PIPE_SLOTS"))
      p->slots = std::max(2, std::min(spmvtk_pipeline::kMaxSlots, std::atoi(e)));
    rt::check(cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking), "pipeline stream");
    for (int k = 0; k < p->split; ++k) {
      rt::check(cudaStreamCreateWithFlags(&p->h2d[k], cudaStreamNonBlocking), "pipeline stream");
      rt::check(cudaStreamCreateWithFlags(&p->d2h[k], cudaStreamNonBlocking), "pipeline stream");
    }
    const std::size_t nx = std::max<std::int64_t>(m->ncols, 1), ny = std::max<std::int64_t>(m->n, 1);
    for (int b = 0; b < p->slots; ++b) {
      rt::check(cudaMalloc(&p->x[b], nx * sizeof(double)), "pipeline x");
      rt::check(cudaMalloc(&p->y[b], ny * sizeof(double)), "pipeline y");
      rt::check(cudaEventCreateWithFlags(&p->comp_done[b], cudaEventDisableTiming), "event");
      for (int k = 0; k < p->split; ++k) {
        rt::check(cudaEventCreateWithFlags(&p->h2d_done[b][k], cudaEventDisableTiming), "event");
        rt::check(cudaEventCreateWithFlags(&p->d2h_done[b][k], cudaEventDisableTiming), "event");
      }
    }
    *out = p.release();
  });
}

spmvtk_status spmvtk_pipeline_submit(spmvtk_pipeline* p, const double* x, double* y) {
  return guarded([&] {
    if (!p || !x || !y) throw Error(ErrorCode::InvalidArgument, "null argument");
    const int b = static_cast<int>(p->count % static_cast<std::uint64_t>(p->slots));
    const std::size_t nx = static_cast<std::size_t>(p->m->ncols);
    const std::size_t ny = static_cast<std::size_t>(p->m->n);
    const int K = p->split;
    // copy-in waits until the SpMV that last read this staging slot is done
    for (int k = 0; k < K; ++k) {
      const std::size_t a = nx * k / K, e = nx * (k + 1) / K;
      rt::check(cudaStreamWaitEvent(p->h2d[k], p->comp_done[b], 0), "pipeline order");
      if (e > a)
        rt::check(cudaMemcpyAsync(p->x[b] + a, x + a, (e - a) * sizeof(double),
                                  cudaMemcpyHostToDevice, p->h2d[k]),
                  "H2D x");
      rt::check(cudaEventRecord(p->h2d_done[b][k], p->h2d[k]), "pipeline event");
      // the SpMV waits for its x and for the copy-out that last read its y slot
      rt::check(cudaStreamWaitEvent(p->comp, p->h2d_done[b][k], 0), "pipeline order");
      rt::check(cudaStreamWaitEvent(p->comp, p->d2h_done[b][k], 0), "pipeline order");
    }
    cudaStream_t saved = rt::stream();
    rt::set_stream(p->comp);
    try {
      dev::spmv_device(*p->m, p->kernel, p->x[b], p->y[b]);
    } catch (...) {
      rt::set_stream(saved);
      throw;
    }
    rt::set_stream(saved);
    rt::check(cudaEventRecord(p->comp_done[b], p->comp), "pipeline event");
    for (int k = 0; k < K; ++k) {
      const std::size_t a = ny * k / K, e = ny * (k + 1) / K;
      rt::check(cudaStreamWaitEvent(p->d2h[k], p->comp_done[b], 0), "pipeline order");
      if (e > a)
        rt::check(cudaMemcpyAsync(y + a, p->y[b] + a, (e - a) * sizeof(double),
                                  cudaMemcpyDeviceToHost, p->d2h[k]),
                  "D2H y");
      rt::check(cudaEventRecord(p->d2h_done[b][k], p->d2h[k]), "pipeline event");
    }
    ++p->count;
  });
}

spmvtk_status spmvtk_pipeline_wait(spmvtk_pipeline* p) {
  return guarded([&] {
    if (!p) throw Error(ErrorCode::InvalidArgument, "null argument");
    for (int k = 0; k < p->split; ++k)
      rt::check(cudaStreamSynchronize(p->h2d[k]), "pipeline wait");
    rt::check(cudaStreamSynchronize(p->comp), "pipeline wait");
    for (int k = 0; k < p->split; ++k)
      rt::check(cudaStreamSynchronize(p->d2h[k]), "pipeline wait");
  });
}

void spmvtk_pipeline_free(spmvtk_pipeline* p) { delete p; }

spmvtk_status spmvtk_bench(const spmvtk_matrix* m, spmvtk_kernel variant, int lanes,
                           int repeats, uint64_t max_bytes, spmvtk_bench_result* out) {
  return guarded([&] {
    need(out, "null output");
    const dev::Matrix& a = crs_of(m);
    if (!valid_kernel(variant)) throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
    at::Timings t = at::bench(a, variant, lanes, repeats, max_bytes);
    at::Metrics cm = at::compute_metrics(t);
    out->t_crs = t.t_crs;
    out->t_ell = t.t_ell;
    out->t_trans = t.t_trans;
    out->sp = cm.sp;
    out->tt = cm.tt;
    out->r = cm.r;
  });
}

spmvtk_status spmvtk_profile_build(const spmvtk_matrix* const* matrices,
                                   const char* const* ids, size_t count,
                                   spmvtk_kernel variant, int lanes, double c, int repeats,
                                   uint64_t max_bytes, const char* machine_label,
                                   spmvtk_profile** out) {
  return guarded([&] {
    if (!matrices || !ids || !out) throw Error(ErrorCode::InvalidArgument, "null argument");
    if (!valid_kernel(variant)) throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
    std::vector<std::pair<std::string, const dev::Matrix*>> set;
    for (size_t i = 0; i < count; ++i) set.emplace_back(ids[i] ? ids[i] : "", &crs_of(matrices[i]));
    auto prof = std::make_unique<spmvtk_profile>();
    prof->p = at::offline_profile(set, variant, lanes, c, repeats, max_bytes,
                                  machine_label ? machine_label : "");
    *out = prof.release();
  });
}

spmvtk_status spmvtk_profile_write(const spmvtk_profile* p, const char* path) {
  return guarded([&] {
    if (!p || !path) throw Error(ErrorCode::InvalidArgument, "null argument");
    std::ofstream f(path);
    if (!f) throw Error(ErrorCode::Io, std::string("cannot open ") + path + " for writing");
    f << at::profile_to_json(p->p) << '\n';
    if (!f) throw Error(ErrorCode::Io, std::string("write failed: ") + path);
  });
}

spmvtk_status spmvtk_profile_read(const char* path, spmvtk_profile** out) {
  return guarded([&] {
    if (!path || !out) throw Error(ErrorCode::InvalidArgument, "null argument");
    std::ifstream f(path);
    if (!f) throw Error(ErrorCode::Io, std::string("cannot open ") + path);
    std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    auto prof = std::make_unique<spmvtk_profile>();
    prof->p = at::profile_from_json(text);
    *out = prof.release();
  });
}

double spmvtk_profile_d_star(const spmvtk_profile* p) { return p ? p->p.d_star : 0.0; }
double spmvtk_profile_c(const spmvtk_profile* p) { return p ? p->p.c : 0.0; }
int spmvtk_profile_lanes(const spmvtk_profile* p) { return p ? p->p.lanes : 0; }
spmvtk_kernel spmvtk_profile_kernel(const spmvtk_profile* p) {
  return p ? p->p.kernel : SPMVTK_KERNEL_CRS;
}
size_t spmvtk_profile_record_count(const spmvtk_profile* p) { return p ? p->p.records.size() : 0; }

spmvtk_status spmvtk_profile_record(const spmvtk_profile* p, size_t index,
                                    spmvtk_record_view* out) {
  return guarded([&] {
    if (!p || !out) throw Error(ErrorCode::InvalidArgument, "null argument");
    if (index >= p->p.records.size())
      throw Error(ErrorCode::InvalidArgument, "record index out of range");
    const at::Record& r = p->p.records[index];
    const double nan = std::numeric_limits<double>::quiet_NaN();
    out->matrix_id = r.matrix_id.c_str();
    out->n = r.n;
    out->nnz = r.nnz;
    out->mu = r.mu;
    out->sigma = r.sigma;
    out->d_mat = r.d_mat;
    out->excluded = r.excluded ? 1 : 0;
    out->exclusion_reason = r.exclusion_reason ? r.exclusion_reason->c_str() : nullptr;
    out->t_crs = r.timings ? r.timings->t_crs : nan;
    out->t_ell = r.timings ? r.timings->t_ell : nan;
    out->t_trans = r.timings ? r.timings->t_trans : nan;
    out->sp = r.metrics ? r.metrics->sp : nan;
    out->tt = r.metrics ? r.metrics->tt : nan;
    out->r = r.metrics ? r.metrics->r : nan;
  });
}

spmvtk_status spmvtk_select(const spmvtk_matrix* m, const spmvtk_profile* p,
                            spmvtk_decision* decision, double* d_mat) {
  return guarded([&] {
    if (!p || !decision) throw Error(ErrorCode::InvalidArgument, "null argument");
    const dev::Matrix& a = crs_of(m);
    // fresh GPU reduction for the on-line phase (autotune.cpp:231-236)
    rt::init();
    rt::Moments mo = rt::row_moments(a.ptr.get(), a.n);
    double dm = rt::stats_from_moments(mo, a.n).d_mat;
    *decision = dm < p->p.d_star ? SPMVTK_USE_ELL : SPMVTK_USE_CRS;
    if (d_mat) *d_mat = dm;
  });
}

// ------------------------------ extensions -------------------------------

void spmvtk_set_stream(void* stream) { rt::set_stream(static_cast<cudaStream_t>(stream)); }
void* spmvtk_get_stream(void) { return rt::stream(); }

spmvtk_status spmvtk_synchronize(void) {
  return guarded([&] { rt::sync(); });
}

spmvtk_status spmvtk_matrix_from_crs(int64_t n, int64_t nnz, const void* row_ptr,
                                     const void* col_idx, const double* values,
                                     int index_width, int index_base, int on_device,
                                     spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = dev::crs_from_arrays(n, nnz, row_ptr, col_idx, values, index_width, index_base,
                                on_device != 0);
  });
}

spmvtk_status spmvtk_matrix_from_crs_block(int64_t nrows, int64_t ncols, int64_t row_offset,
                                           int64_t nnz, const void* row_ptr, const void* col_idx,
                                           const double* values, int index_width, int index_base,
                                           int on_device, spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = dev::crs_block_from_arrays(nrows, ncols, row_offset, nnz, row_ptr, col_idx, values,
                                      index_width, index_base, on_device != 0);
  });
}

spmvtk_status spmvtk_matrix_to_crs(const spmvtk_matrix* m, spmvtk_matrix** out) {
  return guarded([&] {
    need(m);
    need(out, "null output");
    *out = dev::to_crs(*m);
  });
}

spmvtk_status spmvtk_matrix_describe(const spmvtk_matrix* m, spmvtk_matrix_desc* out) {
  return guarded([&] {
    need(m);
    need(out);
    out->format = m->format;
    out->ordering = m->ordering;
    out->n = m->n;
    out->nnz = m->nnz;
    out->band_count = m->band_count;
    out->ld = m->ld;
    out->device_bytes = m->device_bytes();
    out->ncols = m->ncols;
    out->row_offset = m->row_offset;
  });
}

spmvtk_status spmvtk_matrix_copy_array(const spmvtk_matrix* m, spmvtk_array which, void* dst,
                                       int64_t capacity, int index_width, int index_base,
                                       int64_t* len) {
  return guarded([&] {
    need(m);
    need(len);
    if (index_base != 0 && index_base != 1)
      throw Error(ErrorCode::InvalidArgument, "index_base must be 0 or 1");
    *len = dev::copy_array(*m, which, dst, capacity, index_width, index_base);
  });
}

spmvtk_status spmvtk_matrix_device_array(const spmvtk_matrix* m, spmvtk_array which, void** ptr,
                                         int64_t* len) {
  return guarded([&] {
    need(m);
    need(ptr);
    std::int64_t l = dev::device_array(*m, which, ptr);
    if (len) *len = l;
  });
}

spmvtk_status spmvtk_spmv_device(const spmvtk_matrix* m, spmvtk_kernel kernel, const double* x,
                                 double* y) {
  return guarded([&] {
    if (!m || ((!x || !y) && m->n > 0)) throw Error(ErrorCode::InvalidArgument, "null argument");
    if (!valid_kernel(kernel)) throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
    dev::spmv_device(*m, kernel, x, y);
  });
}

spmvtk_status spmvtk_matrix_row_stats(const spmvtk_matrix* m, spmvtk_row_stats* out) {
  return guarded([&] {
    need(out, "null output");
    const dev::Matrix& a = crs_of(m);
    rt::Moments mo = dev::crs_moments(a);
    out->n = a.n;
    out->nnz = a.nnz;
    out->max_row = static_cast<int64_t>(mo.max);
    rt::RowStatsD s = rt::stats_from_moments(mo, a.n);
    out->mu = s.mu;
    out->sigma = s.sigma;
    out->d_mat = s.d_mat;
  });
}

spmvtk_status spmvtk_gen_baseline(int config, int64_t param, double dparam, uint64_t seed,
                                  spmvtk_matrix** out) {
  return guarded([&] {
    need(out, "null output");
    *out = upload(gen::baseline(config, param, dparam, seed));
  });
}

struct spmvtk_host_crs {
  gen::HostCrs h;
};

spmvtk_status spmvtk_gen_baseline_host(int config, int64_t param, double dparam, uint64_t seed,
                                       spmvtk_host_crs** out, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    need(out, "null output");
    auto h = std::make_unique<spmvtk_host_crs>();
    h->h = gen::baseline(config, param, dparam, seed);
    if (n) *n = h->h.n;
    if (nnz) *nnz = h->h.nnz();
    *out = h.release();
  });
}

spmvtk_status spmvtk_host_crs_export(const spmvtk_host_crs* hc, int64_t* row_ptr,
                                     int64_t* col_idx, double* values, int index_base) {
  return guarded([&] {
    need(hc);
    const gen::HostCrs& h = hc->h;
    const std::int64_t shift = index_base - h.base;
    if (row_ptr)
      for (std::int64_t i = 0; i <= h.n; ++i)
        row_ptr[i] = (h.wide() ? h.row_ptr[i] : h.row_ptr32[i]) + shift;
    if (col_idx)
      for (std::int64_t p = 0; p < h.nnz(); ++p)
        col_idx[p] = (h.wide() ? h.col_idx[p] : h.col32[p]) + shift;
    if (values) std::memcpy(values, h.values.data(), h.values.size() * sizeof(double));
  });
}

void spmvtk_host_crs_free(spmvtk_host_crs* h) { delete h; }

spmvtk_status spmvtk_read_matrix_market_host(const char* path, spmvtk_host_crs** out, int64_t* n,
                                             int64_t* nnz) {
  return guarded([&] {
    need(path);
    need(out, "null output");
    auto h = std::make_unique<spmvtk_host_crs>();
    h->h = mm::read(path);
    if (n) *n = h->h.n;
    if (nnz) *nnz = h->h.nnz();
    *out = h.release();
  });
}

spmvtk_status spmvtk_matrix_from_host_crs(const spmvtk_host_crs* h, spmvtk_matrix** out) {
  return guarded([&] {
    need(h);
    need(out, "null output");
    *out = upload(h->h);
  });
}

spmvtk_status spmvtk_matrix_copy_ell_bands(const spmvtk_matrix* m, int64_t k0, int64_t k1,
                                           double* values, int64_t* col_idx, int index_base) {
  return guarded([&] {
    need(m);
    if (index_base != 0 && index_base != 1)
      throw Error(ErrorCode::InvalidArgument, "index_base must be 0 or 1");
    dev::copy_ell_bands(*m, k0, k1, values, col_idx, index_base);
  });
}

// ---- multi-GPU (dist.cpp) ---------------------------------------------------
spmvtk_status spmvtk_dist_unique_id(unsigned char* id) {
  return guarded([&] {
    need(id, "null output");
    spmvtk::dist::unique_id(id);
  });
}

spmvtk_status spmvtk_dist_init(int rank, int world, const unsigned char* id, spmvtk_dist** out) {
  return guarded([&] {
    need(id);
    need(out, "null output");
    *out = spmvtk::dist::init(rank, world, id);
  });
}

void spmvtk_dist_free(spmvtk_dist* d) { spmvtk::dist::destroy(d); }

spmvtk_status spmvtk_partition_rows(const int64_t* row_ptr, int64_t n, int world, int64_t* begin) {
  return guarded([&] {
    need(row_ptr);
    need(begin, "null output");
    if (n < 0) throw Error(ErrorCode::InvalidArgument, "negative dimension");
    const std::vector<std::int64_t> b = gen::partition_rows(row_ptr, n, world);
    std::copy(b.begin(), b.end(), begin);
  });
}

spmvtk_status spmvtk_matrix_distribute(const spmvtk_dist* d, int64_t n, const void* row_ptr,
                                       const void* col_idx, const double* values,
                                       int index_width, int index_base, spmvtk_matrix** out) {
  return guarded([&] {
    need(d);
    need(row_ptr);
    need(out, "null output");
    if (index_width != 4 && index_width != 8)
      throw Error(ErrorCode::InvalidArgument, "index width must be 4 or 8");
    if (n < 0) throw Error(ErrorCode::InvalidArgument, "negative dimension");
    std::vector<std::int64_t> rp(static_cast<std::size_t>(n) + 1);
    for (std::int64_t i = 0; i <= n; ++i)
      rp[static_cast<std::size_t>(i)] =
          index_width == 8 ? static_cast<const std::int64_t*>(row_ptr)[i]
                           : static_cast<const std::int32_t*>(row_ptr)[i];
    const int rank = spmvtk::dist::rank_of(*d);
    const std::vector<std::int64_t> b = gen::partition_rows(rp.data(), n, spmvtk::dist::world_of(*d));
    const std::int64_t r0 = b[static_cast<std::size_t>(rank)],
                       r1 = b[static_cast<std::size_t>(rank) + 1];
    // the block's pointers relative to its first entry (in the caller's base
    // and width, like its column indices)
    const std::int64_t e0 = rp[static_cast<std::size_t>(r0)] - index_base;
    const std::int64_t cnt = rp[static_cast<std::size_t>(r1)] - rp[static_cast<std::size_t>(r0)];
    std::vector<std::int64_t> lrp(static_cast<std::size_t>(r1 - r0) + 1);
    for (std::int64_t i = r0; i <= r1; ++i)
      lrp[static_cast<std::size_t>(i - r0)] = rp[static_cast<std::size_t>(i)] - e0;
    std::vector<std::int32_t> lrp32;
    if (index_width == 4) lrp32.assign(lrp.begin(), lrp.end());
    const char* ci = static_cast<const char*>(col_idx) + e0 * index_width;
    *out = dev::crs_block_from_arrays(
        r1 - r0, n, r0, cnt,
        index_width == 8 ? static_cast<const void*>(lrp.data()) : static_cast<const void*>(lrp32.data()),
        cnt ? ci : nullptr, cnt ? values + e0 : nullptr, index_width, index_base, false);
  });
}

spmvtk_status spmvtk_gen_baseline_shard_host(int config, int64_t param, double dparam,
                                             uint64_t seed, int rank, int world,
                                             spmvtk_host_crs** out, int64_t* rows,
                                             int64_t* row_offset, int64_t* ncols) {
  return guarded([&] {
    need(out, "null output");
    auto h = std::make_unique<spmvtk_host_crs>();
    h->h = gen::baseline_shard(config, param, dparam, seed, rank, world);
    if (rows) *rows = h->h.n;
    if (row_offset) *row_offset = h->h.row_offset;
    if (ncols) *ncols = h->h.ncols < 0 ? h->h.n : h->h.ncols;
    *out = h.release();
  });
}

spmvtk_status spmvtk_gen_baseline_shard(const spmvtk_dist* d, int config, int64_t param,
                                        double dparam, uint64_t seed, spmvtk_matrix** out) {
  return guarded([&] {
    need(d);
    need(out, "null output");
    *out = upload(gen::baseline_shard(config, param, dparam, seed, spmvtk::dist::rank_of(*d),
                                      spmvtk::dist::world_of(*d)));
  });
}

spmvtk_status spmvtk_dist_spmv_iterate(const spmvtk_dist* d, const spmvtk_matrix* m,
                                       spmvtk_kernel kernel, double* x, int64_t steps,
                                       double* seconds) {
  return guarded([&] {
    need(d);
    need(m);
    if (m->ncols > 0) need(x);
    const double s = spmvtk::dist::iterate(*d, *m, kernel, x, steps);
    if (seconds) *seconds = s;
  });
}

struct spmvtk_dist_push {
  spmvtk::dist::Push* p = nullptr;
  ~spmvtk_dist_push() { spmvtk::dist::push_free(p); }
};

spmvtk_status spmvtk_dist_push_create(const spmvtk_dist* d, const spmvtk_matrix* shard,
                                      spmvtk_kernel kernel, int sparse, spmvtk_dist_push** out) {
  return guarded([&] {
    need(d);
    need(shard);
    need(out, "null output");
    auto h = std::make_unique<spmvtk_dist_push>();
    h->p = spmvtk::dist::push_create(*d, *shard, kernel, sparse != 0);
    *out = h.release();
  });
}

spmvtk_status spmvtk_dist_push_iterate(spmvtk_dist_push* p, double* x, int64_t steps,
                                       double* seconds) {
  return guarded([&] {
    need(p);
    need(x);
    const double s = spmvtk::dist::push_iterate(*p->p, x, steps);
    if (seconds) *seconds = s;
  });
}

void spmvtk_dist_push_free(spmvtk_dist_push* p) { delete p; }

spmvtk_status spmvtk_gen_vector(int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    need(out, "null output");
    gen::vector_u11(n, seed, out);
  });
}

spmvtk_status spmvtk_conversion_bytes(const spmvtk_matrix* m, spmvtk_format to,
                                      uint64_t* reference_estimate, uint64_t* device_bytes) {
  return guarded([&] {
    const dev::Matrix& a = crs_of(m);
    if (!valid_format(to)) throw Error(ErrorCode::InvalidArgument, "unknown target format");
    if (reference_estimate) *reference_estimate = dev::reference_ell_estimate(a);
    if (device_bytes) *device_bytes = dev::device_bytes_for(a, to);
  });
}

spmvtk_status spmvtk_transform_kernel_seconds(const spmvtk_matrix* m, spmvtk_format to,
                                              int repeats, double* seconds) {
  return guarded([&] {
    need(seconds);
    const dev::Matrix& a = crs_of(m);
    if (!valid_format(to)) throw Error(ErrorCode::InvalidArgument, "unknown target format");
    *seconds = dev::transform_kernel_seconds(a, to, repeats);
  });
}

// ---- multi-GPU push exchange (spmvtk.h) -----------------------------------
static_assert(sizeof(cudaIpcMemHandle_t) == SPMVTK_IPC_HANDLE_BYTES, "IPC handle size");

spmvtk_status spmvtk_ipc_alloc(uint64_t bytes, void** dev_ptr, void* handle) {
  return guarded([&] {
    need(dev_ptr, "null output");
    need(handle, "null handle buffer");
    rt::init();
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, static_cast<std::size_t>(bytes));
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw Error(ErrorCode::MemoryLimit, "IPC buffer: device allocation of " +
                                              std::to_string(bytes) + " bytes failed");
    }
    rt::check(e, "IPC buffer");
    rt::check(cudaMemset(p, 0, static_cast<std::size_t>(bytes)), "IPC buffer zero");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      rt::check(e, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle, &h, sizeof(h));
    *dev_ptr = p;
  });
}

spmvtk_status spmvtk_ipc_free(void* dev_ptr) {
  return guarded([&] {
    if (dev_ptr) rt::check(cudaFree(dev_ptr), "IPC buffer free");
  });
}

spmvtk_status spmvtk_ipc_open(const void* handle, void** dev_ptr) {
  return guarded([&] {
    need(handle, "null handle");
    need(dev_ptr, "null output");
    rt::init();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    rt::check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess),
              "cudaIpcOpenMemHandle");
  });
}

spmvtk_status spmvtk_ipc_close(void* dev_ptr) {
  return guarded([&] {
    if (dev_ptr) rt::check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  });
}

spmvtk_status spmvtk_spmv_device_push(const spmvtk_matrix* m, spmvtk_kernel kernel,
                                      const double* x, const spmvtk_push* push,
                                      const spmvtk_push_sync* sync) {
  return guarded([&] {
    if (!m || !push || (!x && m->n > 0)) throw Error(ErrorCode::InvalidArgument, "null argument");
    dev::spmv_device_push(*m, kernel, x, *push, sync);
  });
}

spmvtk_status spmvtk_flags_signal(const spmvtk_flag_targets* targets, uint64_t value) {
  return guarded([&] {
    need(targets, "null targets");
    rt::check_launch(spmvtk_k_flags_signal(targets, value, rt::stream()), "flags signal");
  });
}

spmvtk_status spmvtk_flags_wait(const uint64_t* flags, int32_t n, uint64_t value,
                                uint64_t timeout_ns, uint32_t* status) {
  return guarded([&] {
    rt::check_launch(spmvtk_k_flags_wait(flags, n, value, timeout_ns, status, rt::stream()),
                     "flags wait");
  });
}

spmvtk_status spmvtk_reserve_device_memory(uint64_t bytes) {
  return guarded([&] {
    rt::set_pool_keep(bytes);
    rt::DevArray<unsigned char> block(static_cast<std::size_t>(bytes), "pool reservation");
    block.release();
    rt::sync();
  });
}

spmvtk_status spmvtk_compute_metrics(double t_crs, double t_ell, double t_trans, double* sp,
                                     double* tt, double* r) {
  return guarded([&] {
    at::Metrics m = at::compute_metrics(at::Timings{t_crs, t_ell, t_trans});
    if (sp) *sp = m.sp;
    if (tt) *tt = m.tt;
    if (r) *r = m.r;
  });
}

spmvtk_status spmvtk_amortization_iterations(double t_crs, double t_ell, double t_trans,
                                             int64_t* k) {
  return guarded([&] {
    need(k);
    auto v = at::amortization(at::Timings{t_crs, t_ell, t_trans});
    *k = v ? *v : -1;
  });
}

double spmvtk_find_d_star(const double* d_mat, const double* r, size_t count, double c) {
  std::vector<std::pair<double, double>> pts;
  for (size_t i = 0; i < count; ++i) pts.emplace_back(d_mat[i], r[i]);
  return at::find_d_star(std::move(pts), c);
}

const char* spmvtk_version(void) { return "spmvtk-b200 0.1 (sm_100a)"; }

}  // extern "C"
