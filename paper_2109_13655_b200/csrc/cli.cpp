// sssvd-gpu: the reference's command-line front end (proj/tools/sssvd.cpp:1-410) over the B200
// library, so a user of `sssvd` finds the same subcommands, flags, files and exit codes:
//
//   solve        --model 1|2 | --input A.mtx, --interval a b, --L --M --N --ell --delta --eps
//                --alpha --seed --threads --est-rcond-identity --est-rcond-exp --mode --normalize
//                --auto-L --out   -> <out>.report.json (schema v1, report_io.hpp:15-88) and
//                <out>.triplets.csv (report_io.hpp:100-113); GPU-only flags: --device, --gram-cap
//   model        --which --rows --cols --model-seed --out   -> <out>.mtx, <out>.truth.csv
//   filter-plot  --interval --transform --N --alpha --sigma-min --sigma-max --points --log --out
//   bench        --threads --no-scaling --model-seed --seed --out   (bench.hpp:60-100)
//   verify       solve's input/param flags + --mode --inject-noise
//
// Exit codes (sssvd.cpp:21-22, 388-408): 0 ok, 2 configuration / input-format errors, 3
// numerical and other runtime errors, 1 failed verify checks; command-line parse errors exit
// with the CLI11 codes the reference's parser uses (104 conversion, 105 validation, 106 missing
// subcommand, 109 unknown argument).
//
// `verify` keeps the reference's solver-side checks (Galerkin identity, moment identity) and
// reports the two that need a dense CPU SVD oracle of A (oracle self-checks, subspace error
// bound) as skipped: the product binary carries no CPU oracle (tests/ hold the parity checks).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "../../include/sssvd_gpu.hpp"

namespace {

namespace gpu = sssvd::gpu;
constexpr int kExitConfig = 2, kExitNumerical = 3;

// ---------------------------------------------------------------------------- minimal JSON
struct Json {
  using Object = std::map<std::string, Json>;   // sorted keys, like nlohmann::json's default
  using Array = std::vector<Json>;
  std::variant<std::nullptr_t, bool, int64_t, double, std::string, Array, Object> v;
  Json() : v(nullptr) {}
  Json(bool b) : v(b) {}
  Json(int x) : v((int64_t)x) {}
  Json(int64_t x) : v(x) {}
  Json(uint64_t x) : v((int64_t)x) {}
  Json(double x) : v(x) {}
  Json(const char* s) : v(std::string(s)) {}
  Json(std::string s) : v(std::move(s)) {}
  Json(Array a) : v(std::move(a)) {}
  Json(Object o) : v(std::move(o)) {}
  Json& operator[](const std::string& k) {
    if (!std::holds_alternative<Object>(v)) v = Object{};
    return std::get<Object>(v)[k];
  }
  static void str(std::ostream& o, const std::string& s) {
    o << '"';
    for (char c : s) {
      if (c == '"' || c == '\\') o << '\\' << c;
      else if (c == '\n') o << "\\n";
      else if ((unsigned char)c < 0x20) { char b[8]; std::snprintf(b, 8, "\\u%04x", c); o << b; }
      else o << c;
    }
    o << '"';
  }
  void dump(std::ostream& o, int indent, int depth = 0) const {
    const std::string pad((depth + 1) * indent, ' '), end(depth * indent, ' ');
    if (std::holds_alternative<std::nullptr_t>(v)) o << "null";
    else if (auto* b = std::get_if<bool>(&v)) o << (*b ? "true" : "false");
    else if (auto* i = std::get_if<int64_t>(&v)) o << *i;
    else if (auto* d = std::get_if<double>(&v)) {
      if (!std::isfinite(*d)) { o << "null"; return; }         // nlohmann writes NaN/Inf as null
      char buf[64];
      auto r = std::to_chars(buf, buf + 64, *d);                // shortest round-trip form
      std::string t(buf, r.ptr);
      if (t.find_first_of(".e") == std::string::npos) t += ".0";
      o << t;
    } else if (auto* s = std::get_if<std::string>(&v)) str(o, *s);
    else if (auto* a = std::get_if<Array>(&v)) {
      if (a->empty()) { o << "[]"; return; }
      o << "[\n";
      for (size_t k = 0; k < a->size(); ++k) {
        o << pad;
        (*a)[k].dump(o, indent, depth + 1);
        o << (k + 1 < a->size() ? ",\n" : "\n");
      }
      o << end << "]";
    } else {
      const auto& ob = std::get<Object>(v);
      if (ob.empty()) { o << "{}"; return; }
      o << "{\n";
      size_t k = 0;
      for (const auto& [key, val] : ob) {
        o << pad;
        str(o, key);
        o << ": ";
        val.dump(o, indent, depth + 1);
        o << (++k < ob.size() ? ",\n" : "\n");
      }
      o << end << "}";
    }
  }
};

// ---------------------------------------------------------------------------- argument parsing
struct CliError {
  int code;
  std::string what;
};

struct Args {
  std::vector<std::string> a;
  size_t i = 0;
  bool more() const { return i < a.size(); }
  const std::string& next(const std::string& flag) {
    if (i >= a.size()) throw CliError{114, flag + ": expected a value"};
    return a[i++];
  }
};

template <typename T>
T parse_num(const std::string& s, const std::string& flag) {
  T out{};
  if constexpr (std::is_floating_point_v<T>) {
    char* end = nullptr;
    out = std::strtod(s.c_str(), &end);
    if (s.empty() || *end != '\0') throw CliError{104, "Could not convert: " + flag + " = " + s};
  } else {
    auto r = std::from_chars(s.data(), s.data() + s.size(), out);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw CliError{104, "Could not convert: " + flag + " = " + s};
  }
  return out;
}

// ---------------------------------------------------------------------------- the problem on the host
struct Problem {
  int64_t rows = 0, cols = 0;   // user orientation
  bool sparse = false;
  std::vector<double> values;   // dense column-major, or CSC values
  std::vector<int64_t> colptr, rowind;
  std::optional<std::vector<double>> truth;
  std::string source;
  double normalized_scale = 0;

  // y = A x (x: cols x k), column-major
  std::vector<double> apply(const std::vector<double>& x, int64_t k) const {
    std::vector<double> y((size_t)rows * k, 0.0);
    for (int64_t c = 0; c < k; ++c)
      for (int64_t j = 0; j < cols; ++j) {
        const double xj = x[(size_t)c * cols + j];
        if (xj == 0.0) continue;
        if (sparse)
          for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) y[(size_t)c * rows + rowind[q]] += values[q] * xj;
        else
          for (int64_t i = 0; i < rows; ++i) y[(size_t)c * rows + i] += values[(size_t)j * rows + i] * xj;
      }
    return y;
  }
  // y = A^T x (x: rows x k)
  std::vector<double> apply_adjoint(const std::vector<double>& x, int64_t k) const {
    std::vector<double> y((size_t)cols * k, 0.0);
    for (int64_t c = 0; c < k; ++c)
      for (int64_t j = 0; j < cols; ++j) {
        double acc = 0.0;
        if (sparse)
          for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) acc += values[q] * x[(size_t)c * rows + rowind[q]];
        else
          for (int64_t i = 0; i < rows; ++i) acc += values[(size_t)j * rows + i] * x[(size_t)c * rows + i];
        y[(size_t)c * cols + j] = acc;
      }
    return y;
  }
  void upload(gpu::Device& dev) const {
    if (sparse)
      dev.set_operator_csc(rows, cols, colptr.data(), rowind.data(), values.data(), (int64_t)values.size());
    else
      dev.set_operator(values.data(), rows, cols, rows);
  }
};

double norm2(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

// normalize_spectrum (problems.hpp:77-105): power iteration on A^T A, A /= sqrt(lambda)
double normalize_spectrum(Problem& p, double tol = 1e-6, int64_t max_iterations = 20000) {
  const int64_t n = std::min(p.rows, p.cols);
  const bool wide = p.rows < p.cols;   // the reference iterates on the stored (rows >= cols) operator
  std::vector<double> v(n, 1.0 / std::sqrt(double(n)));
  for (int64_t i = 0; i < n; ++i) v[i] += 0.01 * std::sin(double(i + 1));
  double nv = norm2(v);
  for (auto& x : v) x /= nv;
  double lambda = 0.0;
  for (int64_t it = 0; it < max_iterations; ++it) {
    std::vector<double> gv = wide ? p.apply(p.apply_adjoint(v, 1), 1) : p.apply_adjoint(p.apply(v, 1), 1);
    lambda = 0.0;
    for (int64_t i = 0; i < n; ++i) lambda += v[i] * gv[i];
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += (gv[i] - lambda * v[i]) * (gv[i] - lambda * v[i]);
    if (std::sqrt(r) <= tol * lambda) break;
    const double norm = norm2(gv);
    if (norm == 0.0) throw std::invalid_argument("normalize_spectrum: zero matrix");
    for (int64_t i = 0; i < n; ++i) v[i] = gv[i] / norm;
  }
  const double scale = std::sqrt(lambda);
  for (auto& x : p.values) x *= 1.0 / scale;
  return scale;
}

Problem model_problem(int which, int64_t rows, int64_t cols, uint64_t seed) {
  Problem p;
  p.rows = rows;
  p.cols = cols;
  p.values.resize((size_t)rows * cols);
  std::vector<double> sigma(cols);
  gpu::check_host(sssvd_build_model(which, rows, cols, seed, p.values.data(), sigma.data()));
  p.truth = sigma;
  p.source = "model" + std::to_string(which);
  return p;
}

// ---------------------------------------------------------------------------- options
struct SolveOptions {
  int model = 0;
  std::string input;
  uint64_t model_seed = 7;
  double a = 0.8, b = 1.2;
  std::string mode = "ss-svd";
  sssvd_config cfg{};
  bool normalize = false;
  long auto_l = 0;
  std::string out = "sssvd";
  int device = 0;
  double inject_noise = 0;
  SolveOptions() {
    sssvd_default_config(&cfg);
  }
};

int parse_mode(const std::string& mode) {
  if (mode == "ss-svd") return SSSVD_MODE_SS_SVD;
  if (mode == "ss-svd-nt") return SSSVD_MODE_SS_SVD_NT;
  if (mode == "naive") return SSSVD_MODE_NAIVE;
  if (mode == "naive-nt") return SSSVD_MODE_NAIVE_NT;
  throw std::runtime_error("--mode: unknown mode " + mode);   // CLI::ValidationError inside the try: exit 3
}
const char* mode_name(int m) {
  static const char* names[] = {"ss-svd", "ss-svd-nt", "naive", "naive-nt"};
  return names[m];
}
bool exp_mode(int m) { return m == SSSVD_MODE_SS_SVD_NT || m == SSSVD_MODE_NAIVE_NT; }

// common solve/verify flags; returns false if the flag is not one of them
bool solve_flag(const std::string& f, Args& args, SolveOptions& o) {
  auto& p = o.cfg.params;
  if (f == "--model") {
    o.model = parse_num<int>(args.next(f), f);
    if (o.model < 1 || o.model > 2) throw CliError{105, "--model: Value " + std::to_string(o.model) + " not in range [1 - 2]"};
  } else if (f == "--input") o.input = args.next(f);
  else if (f == "--model-seed") o.model_seed = parse_num<uint64_t>(args.next(f), f);
  else if (f == "--interval") {
    o.a = parse_num<double>(args.next(f), f);
    o.b = parse_num<double>(args.next(f), f);
  } else if (f == "--L") p.block_size = parse_num<int64_t>(args.next(f), f);
  else if (f == "--M") p.moment_degree = parse_num<int64_t>(args.next(f), f);
  else if (f == "--N") p.quadrature_count = parse_num<int64_t>(args.next(f), f);
  else if (f == "--ell") p.refinement_steps = parse_num<int64_t>(args.next(f), f);
  else if (f == "--delta") p.lowrank_threshold = parse_num<double>(args.next(f), f);
  else if (f == "--eps") p.spurious_threshold = parse_num<double>(args.next(f), f);
  else if (f == "--alpha") o.cfg.aspect = parse_num<double>(args.next(f), f);
  else if (f == "--seed") p.seed = parse_num<uint64_t>(args.next(f), f);
  else if (f == "--threads") o.cfg.threads = parse_num<int>(args.next(f), f);
  else if (f == "--est-rcond-identity") o.cfg.estimator_rcond_identity = parse_num<double>(args.next(f), f);
  else if (f == "--est-rcond-exp") o.cfg.estimator_rcond_exp = parse_num<double>(args.next(f), f);
  else if (f == "--mode") o.mode = args.next(f);
  else if (f == "--device") o.device = parse_num<int>(args.next(f), f);
  else if (f == "--gram-cap") o.cfg.gram_cap = parse_num<int64_t>(args.next(f), f);
  else return false;
  return true;
}

Problem load_problem(const SolveOptions& o) {
  if ((o.model == 0) == o.input.empty()) throw std::runtime_error("input: give exactly one of --model or --input");
  if (o.model != 0) return model_problem(o.model, 1000, 200, o.model_seed);
  gpu::MarketMatrix m = gpu::read_matrix_market(o.input);
  Problem p;
  p.rows = m.rows;
  p.cols = m.cols;
  p.sparse = m.sparse;
  p.values = std::move(m.values);
  p.colptr = std::move(m.colptr);
  p.rowind = std::move(m.rowind);
  p.source = o.input;
  return p;
}

// host-side configuration checks in the reference's order (ContourRule, then SsParams::validate),
// so configuration errors exit 2 before any GPU work
void validate_config(const sssvd_config& cfg, int64_t n) {
  const int tf = exp_mode(cfg.mode) ? SSSVD_TRANSFORM_EXP : SSSVD_TRANSFORM_IDENTITY;
  const sssvd_status st = sssvd_contour(cfg.interval_a, cfg.interval_b, cfg.params.quadrature_count, cfg.aspect, tf,
                                        nullptr, nullptr, nullptr);
  if (st == SSSVD_E_DOMAIN) throw std::domain_error("ContourRule: Exp transform requires a > 0");
  if (st != SSSVD_OK) throw std::invalid_argument("ContourRule: need 0 <= a < b, even N >= 4, aspect in (0,1]");
  if (sssvd_validate_params(&cfg.params, n) != SSSVD_OK)
    throw std::invalid_argument("SsParams: invalid parameters (L*M <= n, even N >= 4, delta in (0,1), eps > 0)");
}

// ---------------------------------------------------------------------------- result access
struct Host {
  sssvd_result_info info{};
  std::string note;
  std::vector<double> sigma, tau, est, exact, galerkin, left, right, blocks;
  std::vector<int32_t> in_interval, spurious;
};

Host fetch(const gpu::Result& r) {
  Host h;
  h.info = r.info();
  h.note = r.note();
  const int64_t t = h.info.count;
  auto copy = [&](int field, void* dst, size_t count) {
    if (count) gpu::check(sssvd_result_copy(r.raw(), field, dst), nullptr);
  };
  h.sigma.resize(t);
  h.tau.resize(t);
  h.est.resize(t);
  h.exact.resize(t);
  h.galerkin.resize(t);
  h.in_interval.resize(t);
  h.spurious.resize(t);
  h.left.resize((size_t)h.info.rows * t);
  h.right.resize((size_t)h.info.cols * t);
  if (!h.info.empty) {
    copy(SSSVD_FIELD_SIGMA, h.sigma.data(), t);
    copy(SSSVD_FIELD_TAU, h.tau.data(), t);
    copy(SSSVD_FIELD_ESTIMATED, h.est.data(), t);
    copy(SSSVD_FIELD_EXACT, h.exact.data(), t);
    copy(SSSVD_FIELD_GALERKIN, h.galerkin.data(), t);
    copy(SSSVD_FIELD_IN_INTERVAL, h.in_interval.data(), t);
    copy(SSSVD_FIELD_SPURIOUS, h.spurious.data(), t);
    copy(SSSVD_FIELD_LEFT, h.left.data(), h.left.size());
    copy(SSSVD_FIELD_RIGHT, h.right.data(), h.right.size());
  }
  if (!h.info.empty) {
    h.blocks.resize((size_t)(h.info.moment_degree + 1) * h.info.n_internal * h.info.block_size);
    copy(SSSVD_FIELD_BLOCKS, h.blocks.data(), h.blocks.size());
  }
  return h;
}

// accuracy_vs_truth (pipeline.hpp:245-272)
struct Accuracy {
  double max_ns = 0, med_ns = 0, max_all = 0, med_all = 0;
};
Accuracy accuracy_vs_truth(const std::vector<double>& truth, const Host& h) {
  std::vector<double> all, ns;
  for (int64_t i = 0; i < h.info.count; ++i) {
    if (!h.in_interval[i]) continue;
    double best = INFINITY;
    for (double t : truth) best = std::min(best, std::abs(t - h.sigma[i]) / t);
    all.push_back(best);
    if (!h.spurious[i]) ns.push_back(best);
  }
  auto median = [](std::vector<double> v) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    const size_t mid = v.size() / 2;
    return v.size() % 2 ? v[mid] : (v[mid - 1] + v[mid]) / 2.0;
  };
  Accuracy a;
  a.max_all = all.empty() ? 0.0 : *std::max_element(all.begin(), all.end());
  a.max_ns = ns.empty() ? 0.0 : *std::max_element(ns.begin(), ns.end());
  a.med_all = median(all);
  a.med_ns = median(ns);
  return a;
}

Json config_json(const sssvd_config& c) {
  Json j;
  j["interval"] = Json::Array{c.interval_a, c.interval_b};
  j["mode"] = mode_name(c.mode);
  j["transform"] = exp_mode(c.mode) ? "exp" : "identity";
  j["L"] = c.params.block_size;
  j["M"] = c.params.moment_degree;
  j["N"] = c.params.quadrature_count;
  j["ell"] = c.params.refinement_steps;
  j["delta"] = c.params.lowrank_threshold;
  j["epsilon"] = c.params.spurious_threshold;
  j["alpha"] = c.aspect;
  j["seed"] = c.params.seed;
  j["threads"] = c.threads;
  return j;
}

// result_to_json (report_io.hpp:36-88)
Json result_json(const sssvd_config& cfg, const Host& h, const std::optional<Accuracy>& acc) {
  Json j;
  j["schema_version"] = 1;
  j["config"] = config_json(cfg);
  j["empty"] = (bool)h.info.empty;
  if (!h.note.empty()) j["note"] = h.note;
  j["input_transposed"] = (bool)h.info.input_transposed;
  j["retained_rank"] = h.info.retained_rank;
  j["rank_deficient_qr"] = (bool)h.info.rank_deficient_qr;
  Json counts;
  counts["candidates"] = h.info.count;
  counts["in_interval"] = h.info.count_in_interval;
  counts["nonspurious_in_interval"] = h.info.count_nonspurious_in_interval;
  counts["interior"] = h.info.count_interior;
  counts["boundary"] = h.info.count_boundary;
  j["counts"] = counts;
  Json t;
  t["steps_1_2"] = h.info.steps_1_2;
  t["step_3"] = h.info.step_3;
  t["step_4"] = h.info.step_4;
  t["step_5"] = h.info.step_5;
  t["postprocess"] = h.info.postprocess;
  t["total"] = h.info.steps_1_2 + h.info.step_3 + h.info.step_4 + h.info.step_5 + h.info.postprocess;
  j["timings"] = t;
  if (h.info.calibration_index >= 0) {
    Json rc;
    rc["index"] = h.info.calibration_index;
    rc["mu"] = h.info.mu;
    j["residual_calibration"] = rc;
  }
  Json::Array trip;
  for (int64_t i = 0; i < h.info.count; ++i) {
    Json e;
    e["sigma"] = h.sigma[i];
    e["in_interval"] = (bool)h.in_interval[i];
    e["spurious"] = (bool)h.spurious[i];
    e["tau"] = h.tau[i];
    e["residual_estimated"] = h.est[i];
    e["galerkin"] = h.galerkin[i];
    e["residual_exact"] = h.exact[i];
    trip.push_back(e);
  }
  j["triplets"] = trip;
  if (acc) {
    Json a;
    a["max_rel_error_nonspurious"] = acc->max_ns;
    a["median_rel_error_nonspurious"] = acc->med_ns;
    a["max_rel_error_all"] = acc->max_all;
    a["median_rel_error_all"] = acc->med_all;
    j["accuracy"] = a;
  }
  return j;
}

// write_triplets_csv (report_io.hpp:100-113)
void write_triplets_csv(const std::string& path, const Host& h) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("write_triplets_csv: cannot open " + path);
  out << std::setprecision(17);
  out << "index,sigma,in_interval,spurious,tau,residual_exact,residual_estimated,galerkin\n";
  for (int64_t i = 0; i < h.info.count; ++i)
    out << i << "," << h.sigma[i] << "," << int(h.in_interval[i]) << "," << int(h.spurious[i]) << "," << h.tau[i]
        << "," << h.exact[i] << "," << h.est[i] << "," << h.galerkin[i] << "\n";
}

void write_json(const std::string& path, const Json& j) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path);
  j.dump(out, 2);
  out << "\n";
}

sssvd_config finish_config(SolveOptions& o, int64_t n) {
  sssvd_config cfg = o.cfg;
  cfg.interval_a = o.a;
  cfg.interval_b = o.b;
  cfg.mode = parse_mode(o.mode);
  validate_config(cfg, n);
  return cfg;
}

// ---------------------------------------------------------------------------- subcommands
int cmd_solve(SolveOptions& o) {
  if (o.auto_l > 0) {   // LM ~ 3t at fixed M = 4 (sssvd.cpp:121-127)
    o.cfg.params.moment_degree = 4;
    o.cfg.params.block_size = std::max<int64_t>(1, (int64_t)std::lround(3.0 * o.auto_l / 4.0));
  }
  Problem p = load_problem(o);
  if (o.normalize && !p.truth) p.normalized_scale = normalize_spectrum(p);
  const sssvd_config cfg = finish_config(o, std::min(p.rows, p.cols));
  gpu::Device dev(o.device);
  p.upload(dev);
  const Host h = fetch(gpu::run_solve(dev, cfg));
  std::optional<Accuracy> acc;
  if (p.truth) acc = accuracy_vs_truth(*p.truth, h);
  Json j = result_json(cfg, h, acc);
  Json mat;
  mat["rows"] = p.rows;
  mat["cols"] = p.cols;
  mat["source"] = p.source;
  if (p.normalized_scale != 0) mat["normalized_scale"] = p.normalized_scale;
  j["matrix"] = mat;
  write_json(o.out + ".report.json", j);
  write_triplets_csv(o.out + ".triplets.csv", h);
  const auto& i = h.info;
  std::cout << "candidates " << i.count << ", in-interval " << i.count_in_interval << ", non-spurious in-interval "
            << i.count_nonspurious_in_interval << " (interior " << i.count_interior << ", boundary "
            << i.count_boundary << ")\n";
  if (acc) std::cout << "max relative error (non-spurious, vs exact spectrum) " << acc->max_ns << "\n";
  if (!h.note.empty()) std::cout << "note: " << h.note << "\n";
  std::cout << "timings [s]: steps 1-2 " << i.steps_1_2 << ", step 3 " << i.step_3 << ", step 4 " << i.step_4
            << ", step 5 " << i.step_5 << ", total " << (i.steps_1_2 + i.step_3 + i.step_4 + i.step_5 + i.postprocess)
            << "\n";
  std::cout << "report written to " << o.out << ".report.json\n";
  return 0;
}

int cmd_model(int which, int64_t rows, int64_t cols, uint64_t seed, const std::string& out) {
  Problem p = model_problem(which, rows, cols, seed);
  gpu::MarketMatrix m;
  m.rows = rows;
  m.cols = cols;
  m.values = p.values;
  gpu::write_matrix_market(out + ".mtx", m, "model " + std::to_string(which) + " seed " + std::to_string(seed));
  std::ofstream truth(out + ".truth.csv");
  truth << std::setprecision(17) << "index,sigma\n";
  for (size_t i = 0; i < p.truth->size(); ++i) truth << i << "," << (*p.truth)[i] << "\n";
  std::cout << "wrote " << out << ".mtx and " << out << ".truth.csv\n";
  return 0;
}

int cmd_filter_plot(double a, double b, const std::string& transform, int64_t n, double aspect, double smin,
                    double smax, int64_t points, bool log_spacing, const std::string& out) {
  const int tf = transform == "exp" ? SSSVD_TRANSFORM_EXP : SSSVD_TRANSFORM_IDENTITY;
  double cr[2];
  const sssvd_status st = sssvd_contour(a, b, n, aspect, tf, nullptr, nullptr, cr);
  if (st == SSSVD_E_DOMAIN) throw std::domain_error("ContourRule: Exp transform requires a > 0");
  if (st != SSSVD_OK) throw std::invalid_argument("ContourRule: need 0 <= a < b, even N >= 4, aspect in (0,1]");
  if (smin <= 0) smin = a > 0 ? a / 100 : b / 1000;
  if (smax <= 0) smax = b * 10;
  if (points < 1) throw std::invalid_argument("filter_profile: need at least one point");
  std::vector<double> grid(points), vals(points);
  if (sssvd_filter_profile(a, b, n, aspect, tf, smin, smax, points, log_spacing, grid.data(), vals.data()) != SSSVD_OK)
    throw std::invalid_argument("filter_profile: need 0 < sigma_min < sigma_max");
  std::ofstream o(out + ".filter.csv");
  if (!o) throw std::runtime_error("write_filter_csv: cannot open " + out + ".filter.csv");
  o << std::setprecision(17);
  o << "# interval=[" << a << "," << b << "] transform=" << (tf == SSSVD_TRANSFORM_EXP ? "exp" : "identity")
    << " N=" << n << " alpha=" << aspect << " center=" << cr[0] << " radius=" << cr[1] << "\n";
  o << "sigma,abs_f\n";
  for (int64_t i = 0; i < points; ++i) o << grid[i] << "," << vals[i] << "\n";
  std::cout << "wrote " << out << ".filter.csv (" << points << " points)\n";
  return 0;
}

// run_default_bench (bench.hpp:60-100) on the GPU
int cmd_bench(int threads, bool scaling, uint64_t model_seed, uint64_t vin_seed, const std::string& out, int device) {
  struct Row {
    std::string label, error;
    int model = 0, mode = 0;
    int64_t rows = 0, cols = 0, L = 0, M = 0, N = 0, ell = 0, rank = 0, t_hat = 0;
    double t[5] = {0, 0, 0, 0, 0};
    double max_rel = 0, max_res = 0;
  };
  std::vector<Row> rows;
  gpu::Device dev(device);
  auto run_row = [&](const std::string& label, int model_id, const Problem& p, sssvd_config cfg) {
    Row r;
    r.label = label;
    r.model = model_id;
    r.mode = cfg.mode;
    r.rows = p.rows;
    r.cols = p.cols;
    r.L = cfg.params.block_size;
    r.M = cfg.params.moment_degree;
    r.N = cfg.params.quadrature_count;
    r.ell = cfg.params.refinement_steps;
    try {
      validate_config(cfg, std::min(p.rows, p.cols));
      p.upload(dev);
      const Host h = fetch(gpu::run_solve(dev, cfg));
      const auto& i = h.info;
      r.t[0] = i.steps_1_2; r.t[1] = i.step_3; r.t[2] = i.step_4; r.t[3] = i.step_5; r.t[4] = i.postprocess;
      r.rank = i.retained_rank;
      r.t_hat = i.count_nonspurious_in_interval;
      r.max_rel = accuracy_vs_truth(*p.truth, h).max_ns;
      for (int64_t k = 0; k < i.count; ++k)
        if (h.in_interval[k] && !h.spurious[k]) r.max_res = std::max(r.max_res, h.exact[k]);
    } catch (const std::exception& e) {
      r.error = e.what();
    }
    rows.push_back(r);
  };
  const int modes[] = {SSSVD_MODE_NAIVE, SSSVD_MODE_NAIVE_NT, SSSVD_MODE_SS_SVD, SSSVD_MODE_SS_SVD_NT};
  for (int model_id = 1; model_id <= 2; ++model_id) {
    const Problem p = model_problem(model_id, 1000, 200, model_seed);
    for (int mode : modes) {
      sssvd_config cfg;
      sssvd_default_config(&cfg);
      cfg.interval_a = model_id == 1 ? 0.8 : 1e-3;
      cfg.interval_b = model_id == 1 ? 1.2 : 1e-1;
      cfg.mode = mode;
      cfg.threads = threads;
      cfg.params.seed = vin_seed;
      run_row("model" + std::to_string(model_id) + "/" + mode_name(mode), model_id, p, cfg);
    }
  }
  if (scaling) {
    const Problem p = model_problem(1, 1000, 600, model_seed);
    for (int64_t block : {15, 30, 60, 120}) {
      sssvd_config cfg;
      sssvd_default_config(&cfg);
      cfg.interval_a = 0.8;
      cfg.interval_b = 1.2;
      cfg.threads = threads;
      cfg.params.block_size = block;
      cfg.params.seed = vin_seed;
      run_row("scaling/L=" + std::to_string(block), 1, p, cfg);
    }
  }
  {
    std::ofstream csv(out + ".bench.csv");
    if (!csv) throw std::runtime_error("write_bench_csv: cannot open " + out + ".bench.csv");
    csv << std::setprecision(17);
    csv << "label,model,mode,rows,cols,L,M,N,ell,steps_1_2,step_3,step_4,step_5,total,retained_rank,t_hat,"
           "max_rel_error,max_residual,error\n";
    for (const auto& r : rows)
      csv << r.label << "," << r.model << "," << mode_name(r.mode) << "," << r.rows << "," << r.cols << "," << r.L
          << "," << r.M << "," << r.N << "," << r.ell << "," << r.t[0] << "," << r.t[1] << "," << r.t[2] << ","
          << r.t[3] << "," << (r.t[0] + r.t[1] + r.t[2] + r.t[3] + r.t[4]) << "," << r.rank << "," << r.t_hat << ","
          << r.max_rel << "," << r.max_res << "," << r.error << "\n";
  }
  Json::Array arr;
  for (const auto& r : rows) {
    Json e;
    e["label"] = r.label;
    e["model"] = r.model;
    e["mode"] = mode_name(r.mode);
    e["rows"] = r.rows;
    e["cols"] = r.cols;
    e["L"] = r.L;
    e["M"] = r.M;
    e["N"] = r.N;
    e["ell"] = r.ell;
    Json t;
    t["steps_1_2"] = r.t[0];
    t["step_3"] = r.t[1];
    t["step_4"] = r.t[2];
    t["step_5"] = r.t[3];
    t["total"] = r.t[0] + r.t[1] + r.t[2] + r.t[3] + r.t[4];
    e["timings"] = t;
    e["retained_rank"] = r.rank;
    e["t_hat"] = r.t_hat;
    e["max_rel_error"] = r.max_rel;
    e["max_residual"] = r.max_res;
    e["error"] = r.error;
    arr.push_back(e);
  }
  Json bj;
  bj["schema_version"] = 1;
  bj["rows"] = arr;
  write_json(out + ".bench.json", bj);
  std::cout << std::left << std::setw(22) << "label" << std::right << std::setw(11) << "steps 1-2" << std::setw(9)
            << "3" << std::setw(9) << "4" << std::setw(9) << "5" << std::setw(10) << "total" << std::setw(6) << "t"
            << std::setw(12) << "error" << std::setw(12) << "residual" << "\n";
  for (const auto& r : rows) {
    if (!r.error.empty()) {
      std::cout << std::left << std::setw(22) << r.label << "FAILED: " << r.error << "\n";
      continue;
    }
    std::cout << std::left << std::setw(22) << r.label << std::right << std::fixed << std::setprecision(3)
              << std::setw(11) << r.t[0] << std::setw(9) << r.t[1] << std::setw(9) << r.t[2] << std::setw(9) << r.t[3]
              << std::setw(10) << (r.t[0] + r.t[1] + r.t[2] + r.t[3] + r.t[4]) << std::setw(6) << r.t_hat
              << std::scientific << std::setprecision(2) << std::setw(12) << r.max_rel << std::setw(12) << r.max_res
              << "\n"
              << std::defaultfloat;
  }
  std::cout << "wrote " << out << ".bench.csv and " << out << ".bench.json\n";
  return 0;
}

// verify (sssvd.cpp:224-305) without the CPU SVD oracle
int cmd_verify(SolveOptions& o) {
  Problem p = load_problem(o);
  if (std::min(p.rows, p.cols) > 2000) {
    std::cout << "verify: oracle cap exceeded (n > 2000), skipped\n";
    return 0;
  }
  const sssvd_config cfg = finish_config(o, std::min(p.rows, p.cols));
  gpu::Device dev(o.device);
  p.upload(dev);
  Host h = fetch(gpu::run_solve(dev, cfg));
  int failures = 0;
  auto check = [&](const std::string& name, bool ok, double measured, double bound) {
    std::cout << (ok ? "PASS" : "FAIL") << "  " << name << "  (measured " << std::scientific << std::setprecision(3)
              << measured << ", bound " << bound << ")\n"
              << std::defaultfloat;
    if (!ok) ++failures;
  };
  std::cout << "SKIP  oracle reconstruction / orthonormality (no CPU SVD oracle in the GPU CLI)\n";
  // ||A||_2 by power iteration (the reference takes it from its oracle SVD)
  Problem scratch = p;
  const double norm_a = normalize_spectrum(scratch, 1e-10);
  if (o.inject_noise > 0) {   // test hook: corrupt the computed left vectors
    std::mt19937_64 gen(12345);
    std::normal_distribution<double> dist;
    for (auto& x : h.left) x += o.inject_noise * dist(gen);
  }
  double worst_galerkin = 0;
  {
    const int64_t t = h.info.count;
    const std::vector<double> av = p.apply(h.right, t);
    for (int64_t i = 0; i < t; ++i) {
      double s = 0;
      for (int64_t r = 0; r < p.rows; ++r) {
        const double d = av[(size_t)i * p.rows + r] - h.sigma[i] * h.left[(size_t)i * p.rows + r];
        s += d * d;
      }
      worst_galerkin = std::max(worst_galerkin, std::sqrt(s));
    }
  }
  check("Galerkin identity", worst_galerkin <= 1e-10 * norm_a, worst_galerkin, 1e-10 * norm_a);
  if (!exp_mode(cfg.mode) && !h.info.empty) {
    // S_k = G^k S_0 on the internal (rows >= cols) operator
    const int64_t n = h.info.n_internal, L = h.info.block_size;
    const bool wide = p.rows < p.cols;
    auto gram_apply = [&](const std::vector<double>& x) {
      return wide ? p.apply(p.apply_adjoint(x, L), L) : p.apply_adjoint(p.apply(x, L), L);
    };
    std::vector<double> power(h.blocks.begin(), h.blocks.begin() + n * L);
    double worst = 0;
    for (int64_t k = 1; k < cfg.params.moment_degree; ++k) {
      power = gram_apply(power);
      double num = 0, den = 0;
      for (int64_t e = 0; e < n * L; ++e) {
        const double d = h.blocks[(size_t)k * n * L + e] - power[e];
        num += d * d;
        den += power[e] * power[e];
      }
      worst = std::max(worst, std::sqrt(num / den));
    }
    check("moment identity S_k = G^k S_0", worst <= 1e-8, worst, 1e-8);
    std::cout << "SKIP  subspace error bound (needs the exact SVD of A: no CPU oracle in the GPU CLI)\n";
  }
  std::cout << (failures == 0 ? "verify: all checks passed\n"
                              : "verify: " + std::to_string(failures) + " check(s) failed\n");
  return failures == 0 ? 0 : 1;
}

void usage() {
  std::cout << "Partial SVD of a real rectangular matrix on a target interval [a,b]\n"
               "via complex-moment contour integration (B200 / sm_100a)\n"
               "Usage: sssvd-gpu SUBCOMMAND [OPTIONS]\n"
               "Subcommands:\n"
               "  solve        compute singular triplets with sigma in [a,b]\n"
               "  model        generate a model problem as .mtx + truth csv\n"
               "  filter-plot  tabulate |f(sigma)| over a sigma grid\n"
               "  bench        timing table over models and modes\n"
               "  verify       invariant checks, nonzero exit on failure\n";
}

int run(int argc, char** argv) {
  Args args;
  for (int i = 1; i < argc; ++i) args.a.push_back(argv[i]);
  if (!args.more()) {
    usage();
    throw CliError{106, "A subcommand is required"};
  }
  const std::string sub = args.next("subcommand");
  if (sub == "--help" || sub == "-h") {
    usage();
    return 0;
  }
  SolveOptions so;
  if (sub == "solve" || sub == "verify") {
    while (args.more()) {
      const std::string f = args.next("");
      if (solve_flag(f, args, so)) continue;
      if (sub == "solve" && f == "--normalize") so.normalize = true;
      else if (sub == "solve" && f == "--auto-L") so.auto_l = parse_num<long>(args.next(f), f);
      else if (sub == "solve" && f == "--out") so.out = args.next(f);
      else if (sub == "verify" && f == "--inject-noise") so.inject_noise = parse_num<double>(args.next(f), f);
      else throw CliError{109, "The following arguments were not expected: " + f};
    }
    return sub == "solve" ? cmd_solve(so) : cmd_verify(so);
  }
  if (sub == "model") {
    int which = 1;
    int64_t rows = 1000, cols = 200;
    uint64_t seed = 7;
    std::string out = "model";
    while (args.more()) {
      const std::string f = args.next("");
      if (f == "--which") {
        which = parse_num<int>(args.next(f), f);
        if (which < 1 || which > 2) throw CliError{105, "--which: Value not in range [1 - 2]"};
      } else if (f == "--rows") rows = parse_num<int64_t>(args.next(f), f);
      else if (f == "--cols") cols = parse_num<int64_t>(args.next(f), f);
      else if (f == "--model-seed") seed = parse_num<uint64_t>(args.next(f), f);
      else if (f == "--out") out = args.next(f);
      else throw CliError{109, "The following arguments were not expected: " + f};
    }
    return cmd_model(which, rows, cols, seed, out);
  }
  if (sub == "filter-plot") {
    double a = 0.8, b = 1.2, aspect = 0.1, smin = 0, smax = 0;
    int64_t n = 32, points = 200;
    bool log_spacing = false;
    std::string transform = "identity", out = "filter";
    while (args.more()) {
      const std::string f = args.next("");
      if (f == "--interval") {
        a = parse_num<double>(args.next(f), f);
        b = parse_num<double>(args.next(f), f);
      } else if (f == "--transform") transform = args.next(f);
      else if (f == "--N") n = parse_num<int64_t>(args.next(f), f);
      else if (f == "--alpha") aspect = parse_num<double>(args.next(f), f);
      else if (f == "--sigma-min") smin = parse_num<double>(args.next(f), f);
      else if (f == "--sigma-max") smax = parse_num<double>(args.next(f), f);
      else if (f == "--points") points = parse_num<int64_t>(args.next(f), f);
      else if (f == "--log") log_spacing = true;
      else if (f == "--out") out = args.next(f);
      else throw CliError{109, "The following arguments were not expected: " + f};
    }
    return cmd_filter_plot(a, b, transform, n, aspect, smin, smax, points, log_spacing, out);
  }
  if (sub == "bench") {
    int threads = 0, device = 0;
    bool no_scaling = false;
    uint64_t mseed = 7, vseed = 42;
    std::string out = "sssvd";
    while (args.more()) {
      const std::string f = args.next("");
      if (f == "--threads") threads = parse_num<int>(args.next(f), f);
      else if (f == "--no-scaling") no_scaling = true;
      else if (f == "--model-seed") mseed = parse_num<uint64_t>(args.next(f), f);
      else if (f == "--seed") vseed = parse_num<uint64_t>(args.next(f), f);
      else if (f == "--out") out = args.next(f);
      else if (f == "--device") device = parse_num<int>(args.next(f), f);
      else throw CliError{109, "The following arguments were not expected: " + f};
    }
    return cmd_bench(threads, !no_scaling, mseed, vseed, out, device);
  }
  throw CliError{109, "The following arguments were not expected: " + sub};
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const CliError& e) {
    std::cerr << e.what << "\n";
    return e.code;
  } catch (const gpu::NumericalError& ex) {
    std::cerr << "numerical failure: " << ex.what() << "\n";
    return kExitNumerical;
  } catch (const gpu::MatrixMarketError& ex) {
    std::cerr << "input error: " << ex.what() << "\n";
    return kExitConfig;
  } catch (const std::invalid_argument& ex) {
    std::cerr << "configuration error: " << ex.what() << "\n";
    return kExitConfig;
  } catch (const std::domain_error& ex) {
    std::cerr << "configuration error: " << ex.what() << "\n";
    return kExitConfig;
  } catch (const std::length_error& ex) {
    std::cerr << "configuration error: " << ex.what() << "\n";
    return kExitConfig;
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return kExitNumerical;
  }
}
