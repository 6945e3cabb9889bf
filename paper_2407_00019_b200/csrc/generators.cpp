// generators.cpp -- matrix generators.
//
// (1) The reference's three generators (gen_banded / gen_skewed /
//     gen_cv_target, /root/reference/proj/src/ingest.cpp:234-316), restated
//     so equal seeds give byte-identical matrices: mt19937_64 raw outputs
//     only, ranges by `rng() % n`, [0,1) by `(rng() >> 11) * 2^-53`
//     (ingest.cpp:38-73, proj/README.md:136-142).
// (2) The five synthetic BASELINE.json workloads, generated
//     on all host cores in fixed row blocks, each block with its own
//     mt19937_64 stream, so the matrix does not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "generators.hpp"
#include "spmvtk/error.hpp"

namespace spmvtk::gen {

namespace {

using Rng = std::mt19937_64;

std::int64_t below(Rng& r, std::int64_t n) {
  return static_cast<std::int64_t>(r() % static_cast<std::uint64_t>(n));
}
double unit01(Rng& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
double signed_unit(Rng& r) { return 2.0 * unit01(r) - 1.0; }

// k distinct values of 1..n ascending (ingest.cpp:51-73: partial
// Fisher-Yates when k*3 >= n, else rejection), same draw sequence.
std::vector<std::int64_t> distinct_sorted(Rng& r, std::int64_t n, std::int64_t k) {
  std::vector<std::int64_t> out;
  out.reserve(static_cast<std::size_t>(k));
  if (k * 3 >= n) {
    std::vector<std::int64_t> pool(static_cast<std::size_t>(n));
    std::iota(pool.begin(), pool.end(), std::int64_t{1});
    for (std::int64_t i = 0; i < k; ++i) {
      std::int64_t j = i + below(r, n - i);
      std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(j)]);
      out.push_back(pool[static_cast<std::size_t>(i)]);
    }
  } else {
    std::unordered_set<std::int64_t> seen;
    seen.reserve(static_cast<std::size_t>(k) * 2);
    while (static_cast<std::int64_t>(out.size()) < k) {
      std::int64_t v = 1 + below(r, n);
      if (seen.insert(v).second) out.push_back(v);
    }
  }
  std::sort(out.begin(), out.end());
  return out;
}

HostCrs from_degrees(const std::vector<std::int64_t>& deg, Rng& r) {
  HostCrs m;
  m.n = static_cast<std::int64_t>(deg.size());
  m.base = 1;
  m.row_ptr.reserve(deg.size() + 1);
  m.row_ptr.push_back(1);
  for (std::int64_t d : deg) {
    for (std::int64_t j : distinct_sorted(r, m.n, d)) {
      m.col_idx.push_back(j);
      m.values.push_back(signed_unit(r));
    }
    m.row_ptr.push_back(static_cast<std::int64_t>(m.values.size()) + 1);
  }
  return m;
}

}  // namespace

HostCrs banded(std::int64_t n, std::int64_t hw) {
  if (n < 1 || hw < 0 || hw >= n)
    throw Error(ErrorCode::InvalidArgument, "gen_banded requires 0 <= half_width < n");
  HostCrs m;
  m.n = n;
  m.base = 1;
  m.row_ptr.push_back(1);
  for (std::int64_t i = 1; i <= n; ++i) {
    for (std::int64_t j = std::max<std::int64_t>(1, i - hw); j <= std::min(n, i + hw); ++j) {
      m.col_idx.push_back(j);
      m.values.push_back(1.0 / static_cast<double>(1 + std::llabs(i - j)));
    }
    m.row_ptr.push_back(static_cast<std::int64_t>(m.values.size()) + 1);
  }
  return m;
}

HostCrs skewed(std::int64_t n, std::int64_t base_deg, std::int64_t heavy_rows,
               std::int64_t heavy_deg, std::uint64_t seed) {
  if (n < 1 || heavy_rows > n)
    throw Error(ErrorCode::InvalidArgument, "heavy_rows must not exceed n");
  if (base_deg >= n || heavy_deg >= n || base_deg < 0 || heavy_deg < 0)
    throw Error(ErrorCode::InvalidArgument, "row degrees must lie in [0, n)");
  Rng r(seed);
  std::vector<std::int64_t> heavy = distinct_sorted(r, n, heavy_rows);
  std::vector<std::int64_t> deg(static_cast<std::size_t>(n), base_deg);
  for (std::int64_t h : heavy) deg[static_cast<std::size_t>(h - 1)] = heavy_deg;
  return from_degrees(deg, r);
}

HostCrs cv_target(std::int64_t n, double mean_deg, double target, std::uint64_t seed) {
  if (n < 1 || mean_deg <= 0.0 || target < 0.0)
    throw Error(ErrorCode::InvalidArgument, "need n >= 1, mean_deg > 0, target_dmat >= 0");
  Rng r(seed);
  if (target == 0.0) {
    std::int64_t d = std::llround(mean_deg);
    if (d < 1 || d > n)
      throw Error(ErrorCode::InvalidArgument, "mean_deg must round into [1, n] for target 0");
    return from_degrees(std::vector<std::int64_t>(static_cast<std::size_t>(n), d), r);
  }
  // two-point distribution: h equal heavy rows, the rest empty; the CV of
  // the row counts is sqrt((n-h)/h) whatever the heavy degree is
  const double t2 = target * target;
  std::int64_t h = std::llround(static_cast<double>(n) / (1.0 + t2));
  h = std::clamp<std::int64_t>(h, 1, n - 1);
  const long long total = std::llround(mean_deg * static_cast<double>(n));
  const long long per = total / h, extra = total % h;
  if (per + (extra > 0 ? 1 : 0) > n) {
    double max_t = std::sqrt(static_cast<double>(n) /
                                 std::ceil(static_cast<double>(total) / static_cast<double>(n)) -
                             1.0);
    throw Error(ErrorCode::InvalidArgument,
                "target D_mat infeasible: rows would need more than n distinct columns; "
                "feasible range is [0, " +
                    std::to_string(max_t) + "]");
  }
  const double got = std::sqrt(static_cast<double>(n - h) / static_cast<double>(h));
  if (std::abs(got - target) > 0.05 * target)
    throw Error(ErrorCode::InvalidArgument, "target D_mat " + std::to_string(target) +
                                                " not reachable within 5% at n = " +
                                                std::to_string(n) + " (closest " +
                                                std::to_string(got) + ")");
  std::vector<std::int64_t> heavy = distinct_sorted(r, n, h);
  std::vector<std::int64_t> deg(static_cast<std::size_t>(n), 0);
  for (long long k = 0; k < h; ++k)
    deg[static_cast<std::size_t>(heavy[static_cast<std::size_t>(k)] - 1)] =
        per + (k < extra ? 1 : 0);
  return from_degrees(deg, r);
}

// ---------------------------------------------------------------------------
// BASELINE workloads
namespace {

constexpr std::int64_t kBlockRows = 16384;

std::uint64_t mix(std::uint64_t z) {  // splitmix64 finaliser
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double normal(Rng& r) {  // Box-Muller, one variate per call
  double u1 = (static_cast<double>(r() >> 11) + 1.0) * 0x1.0p-53;  // (0,1]
  double u2 = unit01(r);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

// Marsaglia-Tsang; shape < 1 via the U^(1/k) boost
double gamma_sample(Rng& r, double k, double theta) {
  double boost = 1.0;
  if (k < 1.0) {
    double u = (static_cast<double>(r() >> 11) + 1.0) * 0x1.0p-53;
    boost = std::pow(u, 1.0 / k);
    k += 1.0;
  }
  const double d = k - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = normal(r);
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    double u = (static_cast<double>(r() >> 11) + 1.0) * 0x1.0p-53;
    if (u < 1.0 - 0.0331 * x * x * x * x) return d * v * theta * boost;
    if (std::log(u) < 0.5 * x * x + d * (1.0 - v + std::log(v))) return d * v * theta * boost;
  }
}

// `len` distinct sorted columns uniform in [lo, hi) (Floyd's algorithm).
void sample_columns(Rng& r, std::int64_t lo, std::int64_t hi, std::int64_t len,
                    std::vector<std::int32_t>& out, std::unordered_set<std::int64_t>& set) {
  const std::int64_t range = hi - lo;
  out.clear();
  if (len >= range) {
    for (std::int64_t c = lo; c < hi; ++c) out.push_back(static_cast<std::int32_t>(c));
    return;
  }
  if (len <= 48) {
    while (static_cast<std::int64_t>(out.size()) < len) {
      std::int32_t c = static_cast<std::int32_t>(lo + below(r, range));
      if (std::find(out.begin(), out.end(), c) == out.end()) out.push_back(c);
    }
  } else {
    set.clear();
    for (std::int64_t j = range - len; j < range; ++j) {
      std::int64_t t = below(r, j + 1);
      if (!set.insert(t).second) set.insert(j);
    }
    for (std::int64_t v : set) out.push_back(static_cast<std::int32_t>(lo + v));
  }
  std::sort(out.begin(), out.end());
}

// Row-block shard being generated (world == 1: the whole matrix).
struct ShardSpec {
  int rank = 0, world = 1;
};
thread_local ShardSpec t_shard;

// Builds a CRS (base 0, int32 indices) from per-block row generators.  For
// a shard (t_shard.world > 1) every row length is drawn (the partition needs
// them) but only the RNG blocks overlapping the shard's rows are filled.
template <typename LenFn, typename RowFn>
HostCrs build_blocked(std::int64_t n, std::uint64_t seed, LenFn&& row_len, RowFn&& fill_row) {
  HostCrs m;
  m.base = 0;
  const std::int64_t blocks = (n + kBlockRows - 1) / kBlockRows;
  std::vector<std::int64_t> len(static_cast<std::size_t>(n));
  unsigned threads = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  auto run = [&](auto&& body) {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (std::int64_t b = t; b < blocks; b += threads) body(b);
      });
    for (auto& th : pool) th.join();
  };
  // pass 1: lengths (own stream per block)
  run([&](std::int64_t b) {
    Rng r(mix(seed ^ (0x1000000ull + static_cast<std::uint64_t>(b))));
    for (std::int64_t i = b * kBlockRows; i < std::min(n, (b + 1) * kBlockRows); ++i)
      len[static_cast<std::size_t>(i)] = row_len(r, i);
  });
  std::vector<std::int64_t> gptr(static_cast<std::size_t>(n) + 1);
  std::int64_t acc = 0;
  for (std::int64_t i = 0; i < n; ++i) {
    gptr[static_cast<std::size_t>(i)] = acc;
    acc += len[static_cast<std::size_t>(i)];
    if (acc >= INT32_MAX) throw Error(ErrorCode::InvalidArgument, "generated nnz exceeds int32");
  }
  gptr[static_cast<std::size_t>(n)] = acc;
  std::int64_t lo = 0, hi = n;
  if (t_shard.world > 1) {
    const std::vector<std::int64_t> part = partition_rows(gptr.data(), n, t_shard.world);
    lo = part[static_cast<std::size_t>(t_shard.rank)];
    hi = part[static_cast<std::size_t>(t_shard.rank) + 1];
  }
  const std::int64_t e0 = gptr[static_cast<std::size_t>(lo)];
  m.n = hi - lo;
  m.ncols = n;
  m.row_offset = lo;
  m.row_ptr32.resize(static_cast<std::size_t>(m.n) + 1);
  for (std::int64_t i = lo; i <= hi; ++i)
    m.row_ptr32[static_cast<std::size_t>(i - lo)] =
        static_cast<std::int32_t>(gptr[static_cast<std::size_t>(i)] - e0);
  const std::int64_t cnt = gptr[static_cast<std::size_t>(hi)] - e0;
  m.col32.resize(static_cast<std::size_t>(cnt));
  m.values.resize(static_cast<std::size_t>(cnt));
  // pass 2: columns and values (second stream per block) of the blocks that
  // hold rows [lo, hi); rows outside are drawn into a scratch row so the
  // stream advances exactly as in the whole-matrix generation
  run([&](std::int64_t b) {
    const std::int64_t b0 = b * kBlockRows, b1 = std::min(n, (b + 1) * kBlockRows);
    if (b1 <= lo || b0 >= hi) return;
    Rng r(mix(seed ^ (0x2000000ull + static_cast<std::uint64_t>(b))));
    std::vector<std::int32_t> cols, skip_c;
    std::vector<double> skip_v;
    std::unordered_set<std::int64_t> set;
    for (std::int64_t i = b0; i < b1; ++i) {
      const std::int64_t L = len[static_cast<std::size_t>(i)];
      if (i >= lo && i < hi) {
        const std::int64_t a = gptr[static_cast<std::size_t>(i)] - e0;
        fill_row(r, i, L, cols, set, m.col32.data() + a, m.values.data() + a);
      } else {
        skip_c.resize(static_cast<std::size_t>(L));
        skip_v.resize(static_cast<std::size_t>(L));
        fill_row(r, i, L, cols, set, skip_c.data(), skip_v.data());
      }
    }
  });
  return m;
}

HostCrs laplace2d(std::int64_t nx) {
  const std::int64_t n = nx * nx;
  HostCrs m;
  m.n = n;
  m.base = 0;
  m.row_ptr32.push_back(0);
  for (std::int64_t iy = 0; iy < nx; ++iy)
    for (std::int64_t ix = 0; ix < nx; ++ix) {
      const std::int64_t i = iy * nx + ix;
      auto push = [&](std::int64_t c, double v) {
        m.col32.push_back(static_cast<std::int32_t>(c));
        m.values.push_back(v);
      };
      if (iy > 0) push(i - nx, -1.0);
      if (ix > 0) push(i - 1, -1.0);
      push(i, 4.0);
      if (ix + 1 < nx) push(i + 1, -1.0);
      if (iy + 1 < nx) push(i + nx, -1.0);
      m.row_ptr32.push_back(static_cast<std::int32_t>(m.values.size()));
    }
  return m;
}

HostCrs stencil27(std::int64_t nx, std::uint64_t seed) {
  const std::int64_t n = nx * nx * nx;
  auto len = [nx](Rng&, std::int64_t i) {
    const std::int64_t ix = i % nx, iy = (i / nx) % nx, iz = i / (nx * nx);
    auto span = [nx](std::int64_t c) { return (c > 0 ? 1 : 0) + 1 + (c + 1 < nx ? 1 : 0); };
    return static_cast<std::int64_t>(span(ix) * span(iy) * span(iz));
  };
  auto fill = [nx](Rng& r, std::int64_t i, std::int64_t, std::vector<std::int32_t>&,
                   std::unordered_set<std::int64_t>&, std::int32_t* col, double* val) {
    const std::int64_t ix = i % nx, iy = (i / nx) % nx, iz = i / (nx * nx);
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const std::int64_t x = ix + dx, y = iy + dy, z = iz + dz;
          if (x < 0 || y < 0 || z < 0 || x >= nx || y >= nx || z >= nx) continue;
          const std::int64_t c = (z * nx + y) * nx + x;
          col[k] = static_cast<std::int32_t>(c);
          val[k] = (c == i) ? 27.0 : normal(r);
          ++k;
        }
  };
  return build_blocked(n, seed, len, fill);
}

template <typename LenFn>
HostCrs random_rows(std::int64_t n, std::uint64_t seed, std::int64_t window, LenFn&& len_fn) {
  auto fill = [n, window](Rng& r, std::int64_t i, std::int64_t len, std::vector<std::int32_t>& cols,
                          std::unordered_set<std::int64_t>& set, std::int32_t* col, double* val) {
    std::int64_t lo = 0, hi = n;
    if (window > 0) {
      lo = std::max<std::int64_t>(0, i - window);
      hi = std::min<std::int64_t>(n, i + window + 1);
    }
    sample_columns(r, lo, hi, len, cols, set);
    for (std::int64_t k = 0; k < len; ++k) {
      col[k] = cols[static_cast<std::size_t>(k)];
      val[k] = normal(r);
    }
  };
  // a row holds at most the distinct columns of its (edge-clipped) window
  auto len_clipped = [n, window, &len_fn](Rng& r, std::int64_t i) {
    const std::int64_t len = len_fn(r, i);
    if (window <= 0) return std::min<std::int64_t>(len, n);
    const std::int64_t range = std::min<std::int64_t>(n, i + window + 1) -
                               std::max<std::int64_t>(0, i - window);
    return std::min<std::int64_t>(len, range);
  };
  return build_blocked(n, seed, len_clipped, fill);
}

}  // namespace

std::vector<std::int64_t> partition_rows(const std::int64_t* row_ptr, std::int64_t n, int world) {
  if (world < 1) throw Error(ErrorCode::InvalidArgument, "world size must be at least 1");
  std::vector<std::int64_t> begin(static_cast<std::size_t>(world) + 1, n);
  const std::int64_t base = row_ptr[0], nnz = row_ptr[n] - base;
  begin[0] = 0;
  for (int k = 1; k < world; ++k) {
    const std::int64_t target = base + nnz * k / world;
    // first row r in [begin[k-1], n] with row_ptr[r] >= target
    std::int64_t lo = begin[static_cast<std::size_t>(k) - 1], hi = n;
    while (lo < hi) {
      const std::int64_t mid = lo + (hi - lo) / 2;
      if (row_ptr[mid] >= target) hi = mid;
      else lo = mid + 1;
    }
    begin[static_cast<std::size_t>(k)] = lo;
  }
  begin[static_cast<std::size_t>(world)] = n;
  return begin;
}

HostCrs baseline_shard(int config, std::int64_t param, double dparam, std::uint64_t seed,
                       int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world)
    throw Error(ErrorCode::InvalidArgument, "rank must lie in [0, world)");
  if (world == 1) return baseline(config, param, dparam, seed);
  if (config == 1) {  // small and RNG-free: generate, then cut
    HostCrs full = baseline(config, param, dparam, seed);
    std::vector<std::int64_t> ptr(full.row_ptr32.begin(), full.row_ptr32.end());
    const auto part = partition_rows(ptr.data(), full.n, world);
    const std::int64_t lo = part[static_cast<std::size_t>(rank)], hi = part[static_cast<std::size_t>(rank) + 1];
    HostCrs m;
    m.base = 0;
    m.n = hi - lo;
    m.ncols = full.n;
    m.row_offset = lo;
    const std::int32_t e0 = full.row_ptr32[static_cast<std::size_t>(lo)];
    for (std::int64_t i = lo; i <= hi; ++i) m.row_ptr32.push_back(full.row_ptr32[static_cast<std::size_t>(i)] - e0);
    m.col32.assign(full.col32.begin() + e0, full.col32.begin() + full.row_ptr32[static_cast<std::size_t>(hi)]);
    m.values.assign(full.values.begin() + e0, full.values.begin() + full.row_ptr32[static_cast<std::size_t>(hi)]);
    return m;
  }
  t_shard = ShardSpec{rank, world};
  try {
    HostCrs m = baseline(config, param, dparam, seed);
    t_shard = ShardSpec{};
    return m;
  } catch (...) {
    t_shard = ShardSpec{};
    throw;
  }
}

HostCrs baseline(int config, std::int64_t param, double dparam, std::uint64_t seed) {
  switch (config) {
    case 1:
      if (param < 2) throw Error(ErrorCode::InvalidArgument, "grid edge must be >= 2");
      return laplace2d(param);
    case 2: {
      if (param < 25) throw Error(ErrorCode::InvalidArgument, "n must be >= 25");
      return random_rows(param, seed, 0, [](Rng& r, std::int64_t) {
        return static_cast<std::int64_t>(8 + r() % 17);  // U{8..24}
      });
    }
    case 3:
      if (param < 2) throw Error(ErrorCode::InvalidArgument, "grid edge must be >= 2");
      return stencil27(param, seed);
    case 4: {
      if (param < 4096) throw Error(ErrorCode::InvalidArgument, "n must be >= 4096");
      // log-normal with E = exp(mu + s^2/2) = 16: mu = ln 16 - 0.72, s = 1.2
      const double mu = std::log(16.0) - 0.72, sg = 1.2;
      return random_rows(param, seed, 0, [mu, sg](Rng& r, std::int64_t) {
        double v = std::exp(mu + sg * normal(r));
        return std::min<std::int64_t>(4096, std::llround(v));
      });
    }
    case 5: {
      if (param < 64 * 32) throw Error(ErrorCode::InvalidArgument, "n must be >= 2048");
      if (dparam < 0) throw Error(ErrorCode::InvalidArgument, "D must be >= 0");
      const std::int64_t window = param / 64;  // columns within +-n/64
      const std::int64_t cap = std::min<std::int64_t>(65537, 2 * window + 1);
      const double d = dparam;
      return random_rows(param, seed, window, [d, cap](Rng& r, std::int64_t) {
        if (d == 0.0) return static_cast<std::int64_t>(32);
        const double k = 1.0 / (d * d), theta = 32.0 * d * d;
        return std::min<std::int64_t>(cap, std::llround(gamma_sample(r, k, theta)));
      });
    }
  }
  throw Error(ErrorCode::InvalidArgument, "unknown BASELINE config " + std::to_string(config));
}

void vector_u11(std::int64_t n, std::uint64_t seed, double* out) {
  Rng r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = signed_unit(r);
}

}  // namespace spmvtk::gen
