// spmvtk -- the command-line front end over the C ABI (spmvtk.h), with the
// reference CLI's subcommands, options, output lines, CSV schemas and exit
// statuses (proj/tools/spmvtk_cli.cpp; SPEC.md CLI section): 0 success,
// 1 usage error, 2 data / validation error, 3 check failure.
//
//   spmvtk info <matrix.mtx> [--csv]
//   spmvtk convert <matrix.mtx> --to coo-row|coo-col|ccs|ell --out <file> [--max-bytes B]
//   spmvtk spmv <matrix.mtx> [--kernel K] [--lanes L] [--x ones|seed:N] [--check] [--max-bytes B]
//   spmvtk bench <matrix.mtx> [--kernel K] [--lanes L] [--repeats R] [--max-bytes B]
//   spmvtk profile <dir | files...> [--kernel K] [--lanes L] [--c C] [--repeats R]
//                  [--max-bytes B] [--out profile.json] [--csv plot.csv] [--label S]
//   spmvtk select <matrix.mtx> --profile <profile.json>
//   spmvtk gen banded <n> <half_width> --out <file>
//   spmvtk gen skewed <n> <base_deg> <heavy_rows> <heavy_deg> [--seed S] --out <file>
//   spmvtk gen cv-target <n> <mean_deg> <target_dmat> [--seed S] --out <file>
//
// Every matrix lives on the GPU (libspmvtk); `lanes` is accepted and
// validated for compatibility and does not change the kernels.
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "spmvtk/spmvtk.h"

namespace fs = std::filesystem;

namespace {

constexpr uint64_t kEllCapDefault = 2ull << 30;

// ---- failures -----------------------------------------------------------------
struct Exit {
  int code;
};

[[noreturn]] void usage_error(const std::string& what) {
  std::fprintf(stderr, "error: %s\n(run 'spmvtk --help' for usage)\n", what.c_str());
  throw Exit{1};
}

int status_exit(spmvtk_status st) {
  return st == SPMVTK_OK ? 0 : st == SPMVTK_ERR_USAGE ? 1 : st == SPMVTK_ERR_CHECK ? 3 : 2;
}

void ok(spmvtk_status st) {
  if (st == SPMVTK_OK) return;
  std::fprintf(stderr, "error: %s\n", spmvtk_last_error());
  throw Exit{status_exit(st)};
}

// ---- owning handles -------------------------------------------------------------
struct Matrix {
  spmvtk_matrix* h = nullptr;
  Matrix() = default;
  explicit Matrix(spmvtk_matrix* p) : h(p) {}
  Matrix(Matrix&& o) noexcept : h(o.h) { o.h = nullptr; }
  Matrix& operator=(Matrix&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~Matrix() { spmvtk_matrix_free(h); }
};

struct Profile {
  spmvtk_profile* h = nullptr;
  ~Profile() { spmvtk_profile_free(h); }
};

Matrix read_mtx(const std::string& path) {
  spmvtk_matrix* m = nullptr;
  ok(spmvtk_read_matrix_market(path.c_str(), &m));
  return Matrix(m);
}

spmvtk_matrix_info info_of(const Matrix& m) {
  spmvtk_matrix_info i{};
  ok(spmvtk_matrix_get_info(m.h, &i));
  return i;
}

std::string stem(const std::string& path) { return fs::path(path).stem().string(); }

// ---- command line -------------------------------------------------------------------
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;

  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& dflt) const {
    auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) usage_error("option " + k + " is required");
    return opt.at(k);
  }
};

// parse the tokens after the (sub)command name: `valued` options take the
// next token, `flags` take none; anything else starting with "--" is an error
Args parse(int argc, char** argv, int first, const std::set<std::string>& valued,
           const std::set<std::string>& flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string t = argv[i];
    if (t.size() > 2 && t[0] == '-' && t[1] == '-') {
      std::string val;
      const auto eq = t.find('=');
      if (eq != std::string::npos) {
        val = t.substr(eq + 1);
        t = t.substr(0, eq);
      }
      if (flags.count(t)) {
        a.flags.insert(t);
      } else if (valued.count(t)) {
        if (eq == std::string::npos) {
          if (i + 1 >= argc) usage_error("option " + t + " needs a value");
          val = argv[++i];
        }
        a.opt[t] = val;
      } else {
        usage_error("unknown option " + t);
      }
    } else {
      a.pos.push_back(t);
    }
  }
  return a;
}

void positional_count(const Args& a, std::size_t lo, std::size_t hi, const char* what) {
  if (a.pos.size() < lo) usage_error(std::string("missing argument: ") + what);
  if (a.pos.size() > hi) usage_error("unexpected argument " + a.pos[hi]);
}

template <typename T>
T number(const std::string& s, const char* what) {
  try {
    std::size_t used = 0;
    T v;
    if constexpr (std::is_floating_point_v<T>) v = static_cast<T>(std::stod(s, &used));
    else if constexpr (std::is_unsigned_v<T>) v = static_cast<T>(std::stoull(s, &used));
    else v = static_cast<T>(std::stoll(s, &used));
    if (used != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    usage_error(std::string("invalid value for ") + what + ": " + s);
  }
}

struct KernelName {
  const char* name;
  spmvtk_kernel k;
  spmvtk_format input;
};
constexpr KernelName kKernels[] = {
    {"crs", SPMVTK_KERNEL_CRS, SPMVTK_FORMAT_CRS},
    {"coo-row", SPMVTK_KERNEL_COO_ROW_OUTER, SPMVTK_FORMAT_COO_ROW},
    {"coo-col", SPMVTK_KERNEL_COO_COL_OUTER, SPMVTK_FORMAT_COO_COL},
    {"ell-inner", SPMVTK_KERNEL_ELL_INNER, SPMVTK_FORMAT_ELL},
    {"ell-outer", SPMVTK_KERNEL_ELL_OUTER, SPMVTK_FORMAT_ELL},
    {"ell-row", SPMVTK_KERNEL_ELL_ROWMAJOR, SPMVTK_FORMAT_ELL_ROWMAJOR},
};

KernelName kernel_named(const std::string& s) {
  for (const auto& k : kKernels)
    if (s == k.name) return k;
  std::fprintf(stderr, "error: unknown kernel \"%s\"\n", s.c_str());
  throw Exit{1};
}

// x = ones, or U(-1,1) from mt19937_64 raw bits (the generators' mapping)
std::vector<double> x_vector(const std::string& spec, int64_t n) {
  std::vector<double> x(static_cast<std::size_t>(n), 1.0);
  if (spec == "ones") return x;
  if (spec.compare(0, 5, "seed:") == 0) {
    std::mt19937_64 g(number<uint64_t>(spec.substr(5), "--x"));
    for (double& v : x) v = 2.0 * (static_cast<double>(g() >> 11) * 0x1.0p-53) - 1.0;
    return x;
  }
  usage_error("--x must be \"ones\" or \"seed:N\"");
}

std::string quoted(const char* s) {
  std::string q = "\"";
  for (; s && *s; ++s) q += (*s == '"') ? std::string("\"\"") : std::string(1, *s);
  return q + "\"";
}

uint64_t max_bytes_of(const Args& a) {
  return a.has("--max-bytes") ? number<uint64_t>(a.opt.at("--max-bytes"), "--max-bytes")
                              : kEllCapDefault;
}

int lanes_of(const Args& a) {
  const int l = a.has("--lanes") ? number<int>(a.opt.at("--lanes"), "--lanes") : 1;
  return l;
}

// ---- subcommands ----------------------------------------------------------------------
int cmd_info(const Args& a) {
  positional_count(a, 1, 1, "matrix");
  Matrix m = read_mtx(a.pos[0]);
  const spmvtk_matrix_info i = info_of(m);
  const std::string id = stem(a.pos[0]);
  if (a.flags.count("--csv")) {
    std::printf("matrix,n,nnz,mu,sigma,d_mat,max_row_entries,ell_bytes_estimate\n");
    std::printf("%s,%" PRId64 ",%" PRId64 ",%.17g,%.17g,%.17g,%" PRId64 ",%" PRIu64 "\n",
                id.c_str(), i.n, i.nnz, i.mu, i.sigma, i.d_mat, i.max_row_entries, i.ell_bytes);
    return 0;
  }
  std::printf("matrix:            %s\n", id.c_str());
  std::printf("n:                 %" PRId64 "\n", i.n);
  std::printf("nnz:               %" PRId64 "\n", i.nnz);
  std::printf("mu:                %.6g\n", i.mu);
  std::printf("sigma:             %.6g\n", i.sigma);
  std::printf("d_mat:             %.6g\n", i.d_mat);
  std::printf("max row entries:   %" PRId64 "\n", i.max_row_entries);
  std::printf("ELL bytes (est.):  %" PRIu64 "\n", i.ell_bytes);
  return 0;
}

int cmd_convert(const Args& a) {
  positional_count(a, 1, 1, "matrix");
  const std::string to = a.need("--to"), out = a.need("--out");
  static const std::map<std::string, spmvtk_format> targets = {
      {"coo-row", SPMVTK_FORMAT_COO_ROW}, {"coo-col", SPMVTK_FORMAT_COO_COL},
      {"ccs", SPMVTK_FORMAT_CCS},         {"ell", SPMVTK_FORMAT_ELL},
      {"ell-row", SPMVTK_FORMAT_ELL_ROWMAJOR}};
  const auto t = targets.find(to);
  if (t == targets.end()) {
    std::fprintf(stderr, "error: unknown target format \"%s\"\n", to.c_str());
    return 1;
  }
  Matrix m = read_mtx(a.pos[0]);
  spmvtk_matrix* c = nullptr;
  ok(spmvtk_matrix_convert(m.h, t->second, max_bytes_of(a), &c));
  Matrix conv(c);
  ok(spmvtk_write_matrix_market(conv.h, out.c_str()));
  if (t->second == SPMVTK_FORMAT_ELL) {
    const spmvtk_matrix_info i = info_of(m);
    const int64_t padding = i.n * i.max_row_entries - i.nnz;
    char line[256];
    std::snprintf(line, sizeof(line),
                  "band_count=%" PRId64 " stored_nnz=%" PRId64 " padding=%" PRId64
                  " bytes=%" PRIu64,
                  i.max_row_entries, i.nnz, padding, i.ell_bytes);
    std::ofstream(out + ".stats") << line << "\n";
    std::printf("ell: %s\n", line);
  }
  std::printf("wrote %s\n", out.c_str());
  return 0;
}

int cmd_spmv(const Args& a) {
  positional_count(a, 1, 1, "matrix");
  const KernelName kn = kernel_named(a.str("--kernel", "crs"));
  const int lanes = lanes_of(a);
  Matrix crs = read_mtx(a.pos[0]);
  const spmvtk_matrix_info i = info_of(crs);
  Matrix conv;
  if (kn.input != SPMVTK_FORMAT_CRS) {
    spmvtk_matrix* c = nullptr;
    ok(spmvtk_matrix_convert(crs.h, kn.input, max_bytes_of(a), &c));
    conv = Matrix(c);
  }
  const spmvtk_matrix* run_on = kn.input == SPMVTK_FORMAT_CRS ? crs.h : conv.h;
  const std::vector<double> x = x_vector(a.str("--x", "ones"), i.n);
  std::vector<double> y(static_cast<std::size_t>(i.n));
  double secs = 0.0;
  ok(spmvtk_spmv(run_on, kn.k, x.data(), i.n, lanes, y.data(), &secs));
  std::printf("kernel=%s lanes=%d wall_seconds=%.9f\n", kn.name, lanes, secs);
  if (!a.flags.count("--check")) return 0;
  // against the CRS product of the same input (spmv_crs, spmv.cpp:64-75)
  std::vector<double> y0(static_cast<std::size_t>(i.n));
  ok(spmvtk_spmv(crs.h, SPMVTK_KERNEL_CRS, x.data(), i.n, 1, y0.data(), nullptr));
  double scale = 0.0, err = 0.0;
  for (double v : y0) scale = std::max(scale, std::fabs(v));
  if (scale == 0.0) scale = 1.0;
  for (std::size_t r = 0; r < y.size(); ++r) err = std::max(err, std::fabs(y[r] - y0[r]) / scale);
  std::printf("check: max relative error %.3e\n", err);
  if (err > 1e-10) {
    std::fprintf(stderr, "error: check failed (tolerance 1e-10)\n");
    return 3;
  }
  return 0;
}

int cmd_bench(const Args& a) {
  positional_count(a, 1, 1, "matrix");
  const KernelName kn = kernel_named(a.str("--kernel", "ell-outer"));
  const int repeats = a.has("--repeats") ? number<int>(a.opt.at("--repeats"), "--repeats") : 9;
  Matrix m = read_mtx(a.pos[0]);
  const spmvtk_matrix_info i = info_of(m);
  const std::string id = stem(a.pos[0]);
  std::printf("matrix_id,d_mat,t_crs,t_ell,t_trans,sp,tt,r,excluded,exclusion_reason\n");
  spmvtk_bench_result r{};
  const spmvtk_status st = spmvtk_bench(m.h, kn.k, lanes_of(a), repeats, max_bytes_of(a), &r);
  if (st == SPMVTK_ERR_MEMORY_LIMIT) {  // an excluded record, not a failure
    std::printf("%s,%.17g,,,,,,,true,%s\n", id.c_str(), i.d_mat,
                quoted(spmvtk_last_error()).c_str());
    return 0;
  }
  ok(st);
  std::printf("%s,%.17g,%.9e,%.9e,%.9e,%.17g,%.17g,%.17g,false,\n", id.c_str(), i.d_mat, r.t_crs,
              r.t_ell, r.t_trans, r.sp, r.tt, r.r);
  return 0;
}

int cmd_profile(const Args& a) {
  if (a.pos.empty()) usage_error("missing argument: matrices");
  std::vector<std::string> files = a.pos;
  if (files.size() == 1 && fs::is_directory(files[0])) {  // every .mtx inside, sorted
    std::vector<std::string> found;
    for (const auto& e : fs::directory_iterator(files[0]))
      if (e.path().extension() == ".mtx") found.push_back(e.path().string());
    std::sort(found.begin(), found.end());
    files.swap(found);
  }
  if (files.empty()) {
    std::fprintf(stderr, "error: no input matrices\n");
    return 2;
  }
  const KernelName kn = kernel_named(a.str("--kernel", "ell-outer"));
  const double c = a.has("--c") ? number<double>(a.opt.at("--c"), "--c") : 1.0;
  const int repeats = a.has("--repeats") ? number<int>(a.opt.at("--repeats"), "--repeats") : 9;
  const std::string out = a.str("--out", "profile.json"), label = a.str("--label", "");
  std::vector<Matrix> mats;
  std::vector<std::string> ids;
  for (const auto& f : files) {
    mats.push_back(read_mtx(f));
    ids.push_back(stem(f));
  }
  std::vector<const spmvtk_matrix*> hs;
  std::vector<const char*> id_ptrs;
  for (std::size_t k = 0; k < mats.size(); ++k) {
    hs.push_back(mats[k].h);
    id_ptrs.push_back(ids[k].c_str());
  }
  Profile p;
  ok(spmvtk_profile_build(hs.data(), id_ptrs.data(), hs.size(), kn.k, lanes_of(a), c, repeats,
                          max_bytes_of(a), label.c_str(), &p.h));
  ok(spmvtk_profile_write(p.h, out.c_str()));
  if (a.has("--csv")) {  // the (d_mat, r) plot of the included records
    std::ofstream csv(a.opt.at("--csv"));
    csv << "matrix_id,d_mat,r\n";
    for (std::size_t k = 0; k < spmvtk_profile_record_count(p.h); ++k) {
      spmvtk_record_view rec{};
      ok(spmvtk_profile_record(p.h, k, &rec));
      if (rec.excluded) continue;
      char buf[96];
      std::snprintf(buf, sizeof(buf), "%.17g,%.17g", rec.d_mat, rec.r);
      csv << rec.matrix_id << ',' << buf << '\n';
    }
  }
  std::printf("d_star=%.17g\n", spmvtk_profile_d_star(p.h));
  std::printf("wrote %s\n", out.c_str());
  return 0;
}

int cmd_select(const Args& a) {
  positional_count(a, 1, 1, "matrix");
  const std::string prof = a.need("--profile");
  Matrix m = read_mtx(a.pos[0]);
  Profile p;
  ok(spmvtk_profile_read(prof.c_str(), &p.h));
  spmvtk_decision d{};
  double d_mat = 0.0;
  ok(spmvtk_select(m.h, p.h, &d, &d_mat));
  std::printf("%s d_mat=%.17g d_star=%.17g\n", d == SPMVTK_USE_ELL ? "UseEll" : "UseCrs", d_mat,
              spmvtk_profile_d_star(p.h));
  return 0;
}

int write_generated(spmvtk_matrix* raw, const std::string& out) {
  Matrix m(raw);
  ok(spmvtk_write_matrix_market(m.h, out.c_str()));
  const spmvtk_matrix_info i = info_of(m);
  std::printf("n=%" PRId64 " nnz=%" PRId64 " mu=%.6g sigma=%.6g d_mat=%.6g\n", i.n, i.nnz, i.mu,
              i.sigma, i.d_mat);
  std::printf("wrote %s\n", out.c_str());
  return 0;
}

int cmd_gen(int argc, char** argv) {
  if (argc < 3) usage_error("gen needs a generator: banded, skewed or cv-target");
  const std::string kind = argv[2];
  const Args a = parse(argc, argv, 3, {"--out", "--seed"}, {});
  const std::string out = a.need("--out");
  const uint64_t seed = a.has("--seed") ? number<uint64_t>(a.opt.at("--seed"), "--seed") : 0;
  spmvtk_matrix* m = nullptr;
  if (kind == "banded") {
    positional_count(a, 2, 2, "n half_width");
    ok(spmvtk_gen_banded(number<int64_t>(a.pos[0], "n"), number<int64_t>(a.pos[1], "half_width"),
                         &m));
  } else if (kind == "skewed") {
    positional_count(a, 4, 4, "n base_deg heavy_rows heavy_deg");
    ok(spmvtk_gen_skewed(number<int64_t>(a.pos[0], "n"), number<int64_t>(a.pos[1], "base_deg"),
                         number<int64_t>(a.pos[2], "heavy_rows"),
                         number<int64_t>(a.pos[3], "heavy_deg"), seed, &m));
  } else if (kind == "cv-target") {
    positional_count(a, 3, 3, "n mean_deg target_dmat");
    ok(spmvtk_gen_cv_target(number<int64_t>(a.pos[0], "n"), number<double>(a.pos[1], "mean_deg"),
                            number<double>(a.pos[2], "target_dmat"), seed, &m));
  } else {
    usage_error("unknown generator \"" + kind + "\"");
  }
  return write_generated(m, out);
}

void print_usage() {
  std::printf(
      "spmvtk -- sparse SpMV toolkit on B200: format conversion, SpMV kernels and\n"
      "run-time transformation auto-tuning (D_mat / R_ell model)\n\n"
      "  info <matrix.mtx> [--csv]\n"
      "  convert <matrix.mtx> --to coo-row|coo-col|ccs|ell|ell-row --out F [--max-bytes B]\n"
      "  spmv <matrix.mtx> [--kernel K] [--lanes L] [--x ones|seed:N] [--check] [--max-bytes B]\n"
      "  bench <matrix.mtx> [--kernel K] [--lanes L] [--repeats R] [--max-bytes B]\n"
      "  profile <dir|files...> [--kernel K] [--lanes L] [--c C] [--repeats R] [--max-bytes B]\n"
      "          [--out profile.json] [--csv plot.csv] [--label S]\n"
      "  select <matrix.mtx> --profile profile.json\n"
      "  gen banded <n> <half_width> --out F\n"
      "  gen skewed <n> <base_deg> <heavy_rows> <heavy_deg> [--seed S] --out F\n"
      "  gen cv-target <n> <mean_deg> <target_dmat> [--seed S] --out F\n\n"
      "kernels: crs coo-row coo-col ell-inner ell-outer ell-row\n"
      "exit: 0 ok, 1 usage, 2 data/validation, 3 check failure\n");
}

int dispatch(int argc, char** argv) {
  if (argc < 2) usage_error("a subcommand is required");
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    print_usage();
    return 0;
  }
  using Handler = std::function<int(const Args&)>;
  struct Spec {
    std::set<std::string> valued, flags;
    Handler run;
  };
  const std::map<std::string, Spec> table = {
      {"info", {{}, {"--csv"}, cmd_info}},
      {"convert", {{"--to", "--out", "--max-bytes"}, {}, cmd_convert}},
      {"spmv", {{"--kernel", "--lanes", "--x", "--max-bytes"}, {"--check"}, cmd_spmv}},
      {"bench", {{"--kernel", "--lanes", "--repeats", "--max-bytes"}, {}, cmd_bench}},
      {"profile",
       {{"--kernel", "--lanes", "--c", "--repeats", "--max-bytes", "--out", "--csv", "--label"},
        {},
        cmd_profile}},
      {"select", {{"--profile"}, {}, cmd_select}},
  };
  if (cmd == "gen") return cmd_gen(argc, argv);
  const auto it = table.find(cmd);
  if (it == table.end()) usage_error("unknown subcommand \"" + cmd + "\"");
  for (int i = 2; i < argc; ++i)
    if (!std::strcmp(argv[i], "-h") || !std::strcmp(argv[i], "--help")) {
      print_usage();
      return 0;
    }
  return it->second.run(parse(argc, argv, 2, it->second.valued, it->second.flags));
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return dispatch(argc, argv);
  } catch (const Exit& e) {
    return e.code;
  }
}
