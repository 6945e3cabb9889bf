// autotune.hpp -- the D_mat / R_ell auto-tuning model on GPU timings.
//
// Host C++ over the device kernels.  Cost model, amortisation, D* and the
// on-line rule restate /root/reference/proj/src/autotune.cpp:36-60,
// :130-158, :231-236 (TT = t_trans / t_crs as implemented there, not the
// paper's printed Eq. 2 -- SURVEY.md §0.7).  Measurements follow the
// reference protocol (autotune.cpp:95-128) with CUDA events for SpMV.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "matrix.hpp"

namespace spmvtk::at {

struct Timings {
  double t_crs = 0, t_ell = 0, t_trans = 0;
};
struct Metrics {
  double sp = 0, tt = 0, r = 0;
};

Metrics compute_metrics(const Timings& t);
std::optional<std::int64_t> amortization(const Timings& t);
double find_d_star(std::vector<std::pair<double, double>> pts, double c);

const char* kernel_name(spmvtk_kernel k);
spmvtk_kernel kernel_from_name(const std::string& s);
spmvtk_format format_for(spmvtk_kernel k);

// One untimed warm-up, then the median of `repeats` CUDA-event timings of
// one SpMV (seconds).  x = ones as in autotune.cpp:183.
double measure_spmv(const dev::Matrix& m, spmvtk_kernel k, int repeats);
// One cold conversion (allocation and the band-count reduction included),
// wall clock around the call plus a stream synchronisation.
std::pair<dev::Matrix*, double> measure_transformation(const dev::Matrix& crs, spmvtk_format to,
                                                       std::uint64_t max_bytes);

struct Record {
  std::string matrix_id;
  std::int64_t n = 0, nnz = 0;
  double mu = 0, sigma = 0, d_mat = 0;
  std::optional<Timings> timings;
  std::optional<Metrics> metrics;
  bool excluded = false;
  std::optional<std::string> exclusion_reason;
};

struct Profile {
  std::string machine_label;
  spmvtk_kernel kernel = SPMVTK_KERNEL_ELL_OUTER;
  int lanes = 1;
  double c = 1.0;
  std::vector<Record> records;
  double d_star = 0.0;
};

// autotune.cpp:160-229
Profile offline_profile(const std::vector<std::pair<std::string, const dev::Matrix*>>& set,
                        spmvtk_kernel variant, int lanes, double c, int repeats,
                        std::uint64_t max_bytes, const std::string& label);

// (t_crs, t_trans, t_ell) for one CRS handle (capi.cpp:260-306)
Timings bench(const dev::Matrix& crs, spmvtk_kernel variant, int lanes, int repeats,
              std::uint64_t max_bytes);

std::string profile_to_json(const Profile& p);
Profile profile_from_json(const std::string& text);

}  // namespace spmvtk::at
