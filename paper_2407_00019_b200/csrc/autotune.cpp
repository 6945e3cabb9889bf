// autotune.cpp -- see autotune.hpp.
#include "autotune.hpp"

#include <json.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>

#include "runtime.hpp"

namespace spmvtk::at {

Metrics compute_metrics(const Timings& t) {
  if (t.t_crs <= 0.0 || t.t_ell <= 0.0 || t.t_trans <= 0.0)
    throw Error(ErrorCode::InvalidArgument, "timings must be positive");
  Metrics m;
  m.sp = t.t_crs / t.t_ell;    // Eq. 1
  m.tt = t.t_trans / t.t_crs;  // Eq. 2 as implemented (autotune.cpp:41)
  m.r = m.sp / m.tt;           // Eq. 3
  return m;
}

std::optional<std::int64_t> amortization(const Timings& t) {
  if (t.t_crs <= 0.0 || t.t_ell <= 0.0 || t.t_trans <= 0.0)
    throw Error(ErrorCode::InvalidArgument, "timings must be positive");
  if (t.t_ell >= t.t_crs) return std::nullopt;
  // least k with t_trans + k t_ell <= k t_crs; start from the closed form
  // and step across the rounding boundary on both sides
  auto ok = [&](std::int64_t k) {
    return t.t_trans + static_cast<double>(k) * t.t_ell <= static_cast<double>(k) * t.t_crs;
  };
  std::int64_t k = static_cast<std::int64_t>(std::ceil(t.t_trans / (t.t_crs - t.t_ell)));
  while (k > 1 && ok(k - 1)) --k;
  while (!ok(k)) ++k;
  return k;
}

double find_d_star(std::vector<std::pair<double, double>> pts, double c) {
  std::sort(pts.begin(), pts.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  double best = 0.0;
  for (std::size_t i = 0; i < pts.size();) {
    std::size_t j = i;
    bool pass = true;
    for (; j < pts.size() && pts[j].first == pts[i].first; ++j) pass = pass && pts[j].second >= c;
    if (!pass) break;  // a failing tie group ends the admissible prefix
    best = pts[i].first;
    i = j;
  }
  return best;
}

const char* kernel_name(spmvtk_kernel k) { return dev::kernel_label(k); }

spmvtk_kernel kernel_from_name(const std::string& s) {
  for (int k = 0; k <= SPMVTK_KERNEL_ELL_ROWMAJOR; ++k)
    if (s == dev::kernel_label(static_cast<spmvtk_kernel>(k))) return static_cast<spmvtk_kernel>(k);
  throw Error(ErrorCode::InvalidArgument, "unknown kernel name: " + s);
}

spmvtk_format format_for(spmvtk_kernel k) {
  switch (k) {
    case SPMVTK_KERNEL_CRS: return SPMVTK_FORMAT_CRS;
    case SPMVTK_KERNEL_COO_ROW_OUTER: return SPMVTK_FORMAT_COO_ROW;
    case SPMVTK_KERNEL_COO_COL_OUTER: return SPMVTK_FORMAT_COO_COL;
    case SPMVTK_KERNEL_ELL_INNER:
    case SPMVTK_KERNEL_ELL_OUTER: return SPMVTK_FORMAT_ELL;
    case SPMVTK_KERNEL_ELL_ROWMAJOR: return SPMVTK_FORMAT_ELL_ROWMAJOR;
  }
  throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
}

namespace {
void fill_ones(double* d, std::int64_t n) {
  std::vector<double> ones(static_cast<std::size_t>(n), 1.0);
  rt::copy_to_device(d, ones.data(), ones.size() * sizeof(double));
  rt::sync();
}
}  // namespace

double measure_spmv(const dev::Matrix& m, spmvtk_kernel k, int repeats) {
  if (repeats < 1) throw Error(ErrorCode::InvalidArgument, "repeats must be at least 1");
  // x spans the columns (a row-block shard reads global columns in
  // [0, ncols)), y the rows
  const std::int64_t nx = std::max<std::int64_t>(std::max(m.ncols, m.n), 1);
  rt::DevArray<double> x(static_cast<std::size_t>(nx), "x");
  rt::DevArray<double> y(static_cast<std::size_t>(std::max<std::int64_t>(m.n, 1)), "y");
  fill_ones(x.get(), nx);
  dev::spmv_device(m, k, x.get(), y.get());  // warm-up, untimed
  rt::sync();
  std::vector<double> samples;
  rt::EventTimer timer;
  for (int r = 0; r < repeats; ++r) {
    timer.start();
    dev::spmv_device(m, k, x.get(), y.get());
    samples.push_back(timer.stop_seconds());
  }
  std::sort(samples.begin(), samples.end());
  const std::size_t mid = samples.size() / 2;
  return samples.size() % 2 ? samples[mid] : 0.5 * (samples[mid - 1] + samples[mid]);
}

std::pair<dev::Matrix*, double> measure_transformation(const dev::Matrix& crs, spmvtk_format to,
                                                       std::uint64_t max_bytes) {
  rt::sync();
  auto t0 = std::chrono::steady_clock::now();
  dev::Matrix* out = dev::convert(crs, to, max_bytes);
  rt::sync();
  auto t1 = std::chrono::steady_clock::now();
  return {out, std::chrono::duration<double>(t1 - t0).count()};
}

Timings bench(const dev::Matrix& crs, spmvtk_kernel variant, int lanes, int repeats,
              std::uint64_t max_bytes) {
  if (crs.format != SPMVTK_FORMAT_CRS)
    throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
  if (variant == SPMVTK_KERNEL_CRS)
    throw Error(ErrorCode::InvalidArgument, "bench variant must be a transformed-format kernel");
  if (lanes < 1) throw Error(ErrorCode::InvalidArgument, "lane count must be at least 1");
  Timings t;
  t.t_crs = measure_spmv(crs, SPMVTK_KERNEL_CRS, repeats);
  auto [conv, t_trans] = measure_transformation(crs, format_for(variant), max_bytes);
  std::unique_ptr<dev::Matrix> owned(conv);
  t.t_trans = t_trans;
  t.t_ell = measure_spmv(*conv, variant, repeats);
  return t;
}

Profile offline_profile(const std::vector<std::pair<std::string, const dev::Matrix*>>& set,
                        spmvtk_kernel variant, int lanes, double c, int repeats,
                        std::uint64_t max_bytes, const std::string& label) {
  if (set.empty()) throw Error(ErrorCode::InvalidArgument, "empty benchmark matrix set");
  if (c <= 0.0) throw Error(ErrorCode::InvalidArgument, "threshold constant must be positive");
  if (variant == SPMVTK_KERNEL_CRS)
    throw Error(ErrorCode::InvalidArgument, "profile kernel must be a transformed-format kernel");
  if (lanes < 1) throw Error(ErrorCode::InvalidArgument, "lane count must be at least 1");
  Profile p;
  p.machine_label = label;
  p.kernel = variant;
  p.lanes = lanes;
  p.c = c;
  for (const auto& [id, mat] : set) {
    if (!mat || mat->format != SPMVTK_FORMAT_CRS)
      throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
    Record rec;
    rec.matrix_id = id;
    rec.n = mat->n;
    rec.nnz = mat->nnz;
    rt::RowStatsD st = rt::stats_from_moments(dev::crs_moments(*mat), mat->n);
    rec.mu = st.mu;
    rec.sigma = st.sigma;
    rec.d_mat = st.d_mat;
    Timings t;
    t.t_crs = measure_spmv(*mat, SPMVTK_KERNEL_CRS, repeats);
    try {
      auto [conv, t_trans] = measure_transformation(*mat, format_for(variant), max_bytes);
      std::unique_ptr<dev::Matrix> owned(conv);
      t.t_trans = t_trans;
      t.t_ell = measure_spmv(*conv, variant, repeats);
      rec.timings = t;
      rec.metrics = compute_metrics(t);
    } catch (const Error& e) {
      if (e.code() != ErrorCode::MemoryLimit) throw;
      rec.excluded = true;
      rec.exclusion_reason = e.what();
    }
    p.records.push_back(std::move(rec));
  }
  std::vector<std::pair<double, double>> pts;
  for (const auto& r : p.records)
    if (!r.excluded && r.metrics) pts.emplace_back(r.d_mat, r.metrics->r);
  p.d_star = find_d_star(std::move(pts), p.c);
  return p;
}

// ---- profile JSON, schema version 1 (autotune.cpp:264-377) ----------------
namespace {
using nlohmann::json;

void only_keys(const json& o, std::initializer_list<const char*> keys, const char* where) {
  for (const auto& item : o.items()) {
    if (std::none_of(keys.begin(), keys.end(), [&](const char* k) { return item.key() == k; }))
      throw Error(ErrorCode::Parse, std::string("unknown key \"") + item.key() + "\" in " + where);
  }
}
double number(const json& o, const char* key, const char* where) {
  if (!o.contains(key) || !o[key].is_number())
    throw Error(ErrorCode::Parse,
                std::string("missing or non-numeric \"") + key + "\" in " + where);
  return o[key].get<double>();
}
}  // namespace

std::string profile_to_json(const Profile& p) {
  json doc;
  doc["version"] = 1;
  doc["machine_label"] = p.machine_label;
  doc["kernel_variant"] = kernel_name(p.kernel);
  doc["lanes"] = p.lanes;
  doc["c"] = p.c;
  doc["d_star"] = p.d_star;
  json recs = json::array();
  for (const Record& r : p.records) {
    json o;
    o["matrix_id"] = r.matrix_id;
    o["n"] = r.n;
    o["nnz"] = r.nnz;
    o["mu"] = r.mu;
    o["sigma"] = r.sigma;
    o["d_mat"] = r.d_mat;
    o["t_crs"] = r.timings ? json(r.timings->t_crs) : json(nullptr);
    o["t_ell"] = r.timings ? json(r.timings->t_ell) : json(nullptr);
    o["t_trans"] = r.timings ? json(r.timings->t_trans) : json(nullptr);
    o["sp"] = r.metrics ? json(r.metrics->sp) : json(nullptr);
    o["tt"] = r.metrics ? json(r.metrics->tt) : json(nullptr);
    o["r"] = r.metrics ? json(r.metrics->r) : json(nullptr);
    o["excluded"] = r.excluded;
    o["exclusion_reason"] = r.exclusion_reason ? json(*r.exclusion_reason) : json(nullptr);
    recs.push_back(std::move(o));
  }
  doc["records"] = std::move(recs);
  return doc.dump(2);  // shortest round-trip doubles
}

Profile profile_from_json(const std::string& text) {
  json doc;
  try {
    doc = json::parse(text);
  } catch (const json::exception& e) {
    throw Error(ErrorCode::Parse, std::string("profile JSON: ") + e.what());
  }
  if (!doc.is_object()) throw Error(ErrorCode::Parse, "profile JSON is not an object");
  only_keys(doc, {"version", "machine_label", "kernel_variant", "lanes", "c", "d_star", "records"},
            "profile");
  if (!doc.contains("version") || doc["version"] != 1)
    throw Error(ErrorCode::Parse, "profile schema version must be 1");
  Profile p;
  if (!doc.contains("machine_label") || !doc["machine_label"].is_string())
    throw Error(ErrorCode::Parse, "missing machine_label");
  p.machine_label = doc["machine_label"].get<std::string>();
  if (!doc.contains("kernel_variant") || !doc["kernel_variant"].is_string())
    throw Error(ErrorCode::Parse, "missing kernel_variant");
  p.kernel = kernel_from_name(doc["kernel_variant"].get<std::string>());
  if (!doc.contains("lanes") || !doc["lanes"].is_number_integer())
    throw Error(ErrorCode::Parse, "missing lanes");
  p.lanes = doc["lanes"].get<int>();
  p.c = number(doc, "c", "profile");
  p.d_star = number(doc, "d_star", "profile");
  if (!doc.contains("records") || !doc["records"].is_array())
    throw Error(ErrorCode::Parse, "missing records array");
  for (const auto& o : doc["records"]) {
    only_keys(o, {"matrix_id", "n", "nnz", "mu", "sigma", "d_mat", "t_crs", "t_ell", "t_trans", "sp",
                  "tt", "r", "excluded", "exclusion_reason"},
              "record");
    Record r;
    if (!o.contains("matrix_id") || !o["matrix_id"].is_string())
      throw Error(ErrorCode::Parse, "record missing matrix_id");
    r.matrix_id = o["matrix_id"].get<std::string>();
    r.n = static_cast<std::int64_t>(number(o, "n", "record"));
    r.nnz = static_cast<std::int64_t>(number(o, "nnz", "record"));
    r.mu = number(o, "mu", "record");
    r.sigma = number(o, "sigma", "record");
    r.d_mat = number(o, "d_mat", "record");
    if (o.contains("t_crs") && o["t_crs"].is_number())
      r.timings = Timings{number(o, "t_crs", "record"), number(o, "t_ell", "record"),
                          number(o, "t_trans", "record")};
    if (o.contains("sp") && o["sp"].is_number())
      r.metrics = Metrics{number(o, "sp", "record"), number(o, "tt", "record"),
                          number(o, "r", "record")};
    if (!o.contains("excluded") || !o["excluded"].is_boolean())
      throw Error(ErrorCode::Parse, "record missing excluded flag");
    r.excluded = o["excluded"].get<bool>();
    if (o.contains("exclusion_reason") && o["exclusion_reason"].is_string())
      r.exclusion_reason = o["exclusion_reason"].get<std::string>();
    p.records.push_back(std::move(r));
  }
  return p;
}

}  // namespace spmvtk::at
