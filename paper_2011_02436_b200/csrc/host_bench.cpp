// Trial protocol and report formats of the reference's benchmark layer (proj/src/bench.cpp,
// include/rbpelm/bench.hpp), so GPU timings come out in the reference's own
// report schema.  Behaviour restated:
//   * one trial (bench.cpp:19-37): total_seconds is the host wall time around train().
//   * run_trials (bench.cpp:93-130): one discarded warm-up trial at the template seed, then
//     `trials` trainings with seed = base + t; min / max / mean / sample stddev of the wall time,
//     mean solve time and mean training accuracy.
//   * sweep_df_splits (:132-153): one TrialStats per split (each in (0, L)), best / worst by mean.
//   * sweep_nodes (:155-181): node counts x strategies; node counts may not exceed the samples.
//   * JSON schema 1 (:183-215): {"schema":1, machine, dataset{name,samples,features,classes},
//     node_counts, split_points, stats[...]} with per-trial records.  The writer here emits
//     sorted keys and two-space indentation; report_from_json(report_to_json(r)) is lossless
//     (doubles are written with 17 significant digits).
//   * emit_report CSV (:217-238) and per-strategy TSV plot series (:240-266).
#include "../../include/rbpelm_b200.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>

namespace rbpelm {

namespace {

// ---------------------------------------------------------------- trials
TrialRecord one_trial(const Dataset& ds, ElmParams params, const SolverStrategy& strategy, std::uint64_t seed) {
  params.seed = seed;
  const auto t0 = std::chrono::steady_clock::now();
  auto result = train(params, ds.x, ds.y, strategy);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const SolveDiagnostics& d = result.second;
  TrialRecord r;
  r.seed = seed;
  r.total_seconds = wall;
  r.solve_seconds = d.solve_seconds;
  r.hidden_seconds = d.hidden_seconds;
  r.accuracy = d.training_accuracy;
  r.rank = d.rank;
  r.rank_known = d.rank_known;
  r.ridge_applied = d.ridge_applied;
  r.fallback_to_direct = d.fallback_to_direct;
  return r;
}

// ---------------------------------------------------------------- JSON value + writer + parser
struct Json {
  enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;  // sorted keys

  static Json num(double v) { Json j; j.kind = Num; j.d = v; return j; }
  static Json integer(long long v) { Json j; j.kind = Int; j.i = v; return j; }
  static Json boolean(bool v) { Json j; j.kind = Bool; j.b = v; return j; }
  static Json str(const std::string& v) { Json j; j.kind = Str; j.s = v; return j; }
  static Json arr() { Json j; j.kind = Arr; return j; }
  static Json obj() { Json j; j.kind = Obj; return j; }

  const Json& at(const std::string& k) const {
    auto it = o.find(k);
    if (kind != Obj || it == o.end()) throw std::runtime_error("report_from_json: missing key '" + k + "'");
    return it->second;
  }
  double as_double() const {
    if (kind == Num) return d;
    if (kind == Int) return static_cast<double>(i);
    throw std::runtime_error("report_from_json: number expected");
  }
  std::size_t as_size() const {
    if (kind == Int && i >= 0) return static_cast<std::size_t>(i);
    throw std::runtime_error("report_from_json: non-negative integer expected");
  }
  bool as_bool() const {
    if (kind == Bool) return b;
    throw std::runtime_error("report_from_json: boolean expected");
  }
  const std::string& as_str() const {
    if (kind == Str) return s;
    throw std::runtime_error("report_from_json: string expected");
  }
};

std::string quote(const std::string& v) {
  std::string out = "\"";
  for (const unsigned char ch : v) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (ch < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", ch);
          out += buf;
        } else {
          out += static_cast<char>(ch);
        }
    }
  }
  return out + "\"";
}

std::string number(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  std::string s = buf;
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";  // keep the value a float
  return s;
}

void write(const Json& j, int indent, std::string& out) {
  const std::string pad(indent * 2, ' '), pad2((indent + 1) * 2, ' ');
  switch (j.kind) {
    case Json::Null: out += "null"; break;
    case Json::Bool: out += j.b ? "true" : "false"; break;
    case Json::Int: out += std::to_string(j.i); break;
    case Json::Num: out += number(j.d); break;
    case Json::Str: out += quote(j.s); break;
    case Json::Arr:
      if (j.a.empty()) { out += "[]"; break; }
      out += "[\n";
      for (std::size_t k = 0; k < j.a.size(); ++k) {
        out += pad2;
        write(j.a[k], indent + 1, out);
        out += k + 1 < j.a.size() ? ",\n" : "\n";
      }
      out += pad + "]";
      break;
    case Json::Obj: {
      if (j.o.empty()) { out += "{}"; break; }
      out += "{\n";
      std::size_t k = 0;
      for (const auto& kv : j.o) {
        out += pad2 + quote(kv.first) + ": ";
        write(kv.second, indent + 1, out);
        out += ++k < j.o.size() ? ",\n" : "\n";
      }
      out += pad + "}";
      break;
    }
  }
}

struct Parser {
  const std::string& t;
  std::size_t p = 0;
  [[noreturn]] void bad(const std::string& what) const {
    throw std::runtime_error("report_from_json: " + what + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < t.size() && t[p] == c) { ++p; return true; }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) bad(std::string("'") + c + "' expected");
  }
  std::string string_lit() {
    ws();
    if (p >= t.size() || t[p] != '"') bad("string expected");
    ++p;
    std::string out;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c != '\\') { out += c; continue; }
      if (p >= t.size()) bad("bad escape");
      const char e = t[p++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'u': {
          if (p + 4 > t.size()) bad("bad \\u escape");
          const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
          p += 4;
          if (cp < 0x80) {
            out += static_cast<char>(cp);
          } else if (cp < 0x800) {
            out += static_cast<char>(0xC0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          } else {
            out += static_cast<char>(0xE0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: bad("bad escape");
      }
    }
    if (p >= t.size()) bad("unterminated string");
    ++p;
    return out;
  }
  Json value() {
    ws();
    if (p >= t.size()) bad("value expected");
    const char c = t[p];
    if (c == '{') {
      ++p;
      Json j = Json::obj();
      if (eat('}')) return j;
      do {
        const std::string k = string_lit();
        expect(':');
        j.o[k] = value();
      } while (eat(','));
      expect('}');
      return j;
    }
    if (c == '[') {
      ++p;
      Json j = Json::arr();
      if (eat(']')) return j;
      do j.a.push_back(value());
      while (eat(','));
      expect(']');
      return j;
    }
    if (c == '"') return Json::str(string_lit());
    if (t.compare(p, 4, "true") == 0) { p += 4; return Json::boolean(true); }
    if (t.compare(p, 5, "false") == 0) { p += 5; return Json::boolean(false); }
    if (t.compare(p, 4, "null") == 0) { p += 4; return Json(); }
    const std::size_t b = p;
    bool real = false;
    while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '-' || t[p] == '+' ||
                            t[p] == '.' || t[p] == 'e' || t[p] == 'E')) {
      real = real || t[p] == '.' || t[p] == 'e' || t[p] == 'E';
      ++p;
    }
    if (b == p) bad("value expected");
    const std::string tok = t.substr(b, p - b);
    char* end = nullptr;
    if (real) {
      const double v = std::strtod(tok.c_str(), &end);
      if (end != tok.c_str() + tok.size()) bad("bad number");
      return Json::num(v);
    }
    const long long v = std::strtoll(tok.c_str(), &end, 10);
    if (end != tok.c_str() + tok.size()) bad("bad number");
    return Json::integer(v);
  }
};

Json stats_json(const TrialStats& s) {
  Json recs = Json::arr();
  for (const TrialRecord& r : s.records) {
    Json jr = Json::obj();
    jr.o["seed"] = Json::integer(static_cast<long long>(r.seed));
    jr.o["total_seconds"] = Json::num(r.total_seconds);
    jr.o["solve_seconds"] = Json::num(r.solve_seconds);
    jr.o["hidden_seconds"] = Json::num(r.hidden_seconds);
    jr.o["accuracy"] = Json::num(r.accuracy);
    jr.o["rank"] = Json::integer(static_cast<long long>(r.rank));
    jr.o["rank_known"] = Json::boolean(r.rank_known);
    jr.o["ridge_applied"] = Json::boolean(r.ridge_applied);
    jr.o["fallback_to_direct"] = Json::boolean(r.fallback_to_direct);
    recs.a.push_back(jr);
  }
  Json j = Json::obj();
  j.o["strategy"] = Json::str(s.strategy);
  j.o["hidden_nodes"] = Json::integer(static_cast<long long>(s.hidden_nodes));
  j.o["trials"] = Json::integer(static_cast<long long>(s.trials));
  j.o["mean_seconds"] = Json::num(s.mean_seconds);
  j.o["min_seconds"] = Json::num(s.min_seconds);
  j.o["max_seconds"] = Json::num(s.max_seconds);
  j.o["stddev_seconds"] = Json::num(s.stddev_seconds);
  j.o["mean_solve_seconds"] = Json::num(s.mean_solve_seconds);
  j.o["mean_accuracy"] = Json::num(s.mean_accuracy);
  j.o["records"] = recs;
  return j;
}

TrialStats stats_from(const Json& j) {
  TrialStats s;
  s.strategy = j.at("strategy").as_str();
  s.hidden_nodes = j.at("hidden_nodes").as_size();
  s.trials = j.at("trials").as_size();
  s.mean_seconds = j.at("mean_seconds").as_double();
  s.min_seconds = j.at("min_seconds").as_double();
  s.max_seconds = j.at("max_seconds").as_double();
  s.stddev_seconds = j.at("stddev_seconds").as_double();
  s.mean_solve_seconds = j.at("mean_solve_seconds").as_double();
  s.mean_accuracy = j.at("mean_accuracy").as_double();
  for (const Json& jr : j.at("records").a) {
    TrialRecord r;
    r.seed = static_cast<std::uint64_t>(jr.at("seed").as_size());
    r.total_seconds = jr.at("total_seconds").as_double();
    r.solve_seconds = jr.at("solve_seconds").as_double();
    r.hidden_seconds = jr.at("hidden_seconds").as_double();
    r.accuracy = jr.at("accuracy").as_double();
    r.rank = jr.at("rank").as_size();
    r.rank_known = jr.at("rank_known").as_bool();
    r.ridge_applied = jr.at("ridge_applied").as_bool();
    r.fallback_to_direct = jr.at("fallback_to_direct").as_bool();
    s.records.push_back(r);
  }
  return s;
}

Json sizes(const std::vector<std::size_t>& v) {
  Json j = Json::arr();
  for (const std::size_t x : v) j.a.push_back(Json::integer(static_cast<long long>(x)));
  return j;
}

}  // namespace

TrialStats run_trials(const Dataset& ds, const ElmParams& params_template, const SolverStrategy& strategy,
                      std::size_t trials) {
  if (trials < 1) throw std::invalid_argument("run_trials: trials must be >= 1");
  one_trial(ds, params_template, strategy, params_template.seed);  // warm-up, discarded
  TrialStats s;
  s.strategy = strategy.describe();
  s.hidden_nodes = params_template.hidden_nodes;
  s.trials = trials;
  for (std::size_t t = 0; t < trials; ++t) s.records.push_back(one_trial(ds, params_template, strategy, params_template.seed + t));
  double sum = 0.0, sum_solve = 0.0, sum_acc = 0.0;
  s.min_seconds = s.max_seconds = s.records.front().total_seconds;
  for (const TrialRecord& r : s.records) {
    sum += r.total_seconds;
    sum_solve += r.solve_seconds;
    sum_acc += r.accuracy;
    s.min_seconds = std::min(s.min_seconds, r.total_seconds);
    s.max_seconds = std::max(s.max_seconds, r.total_seconds);
  }
  const double n = static_cast<double>(trials);
  s.mean_seconds = sum / n;
  s.mean_solve_seconds = sum_solve / n;
  s.mean_accuracy = sum_acc / n;
  if (trials > 1) {
    double ss = 0.0;
    for (const TrialRecord& r : s.records) ss += (r.total_seconds - s.mean_seconds) * (r.total_seconds - s.mean_seconds);
    s.stddev_seconds = std::sqrt(ss / (n - 1.0));
  }
  return s;
}

SweepResult sweep_df_splits(const Dataset& ds, const ElmParams& params_template,
                            const std::vector<std::size_t>& split_points, std::size_t trials) {
  if (split_points.empty()) throw std::invalid_argument("sweep_df_splits: no split points");
  for (const std::size_t sp : split_points)
    if (sp < 1 || sp >= params_template.hidden_nodes)
      throw std::invalid_argument("sweep_df_splits: split " + std::to_string(sp) + " outside (0, " +
                                  std::to_string(params_template.hidden_nodes) + ")");
  SweepResult r;
  for (const std::size_t sp : split_points)
    r.stats.push_back(run_trials(ds, params_template, SolverStrategy::df_split(sp), trials));
  for (std::size_t i = 1; i < r.stats.size(); ++i) {
    if (r.stats[i].mean_seconds < r.stats[r.best_index].mean_seconds) r.best_index = i;
    if (r.stats[i].mean_seconds > r.stats[r.worst_index].mean_seconds) r.worst_index = i;
  }
  return r;
}

BenchmarkReport sweep_nodes(const Dataset& ds, const ElmParams& params_template,
                            const std::vector<std::size_t>& node_counts,
                            const std::vector<SolverStrategy>& strategies, std::size_t trials,
                            const std::string& machine, const std::string& dataset_name) {
  if (node_counts.empty() || strategies.empty())
    throw std::invalid_argument("sweep_nodes: need at least one node count and one strategy");
  for (const std::size_t l : node_counts)
    if (l > ds.samples())
      throw std::invalid_argument("sweep_nodes: node count " + std::to_string(l) + " exceeds the dataset's " +
                                  std::to_string(ds.samples()) + " samples");
  BenchmarkReport rep;
  rep.machine = machine;
  rep.dataset = {dataset_name, ds.samples(), ds.features(), ds.classes()};
  rep.node_counts = node_counts;
  for (const std::size_t l : node_counts) {
    ElmParams p = params_template;
    p.hidden_nodes = l;
    for (const SolverStrategy& st : strategies) rep.stats.push_back(run_trials(ds, p, st, trials));
  }
  return rep;
}

std::string report_to_json(const BenchmarkReport& report) {
  Json j = Json::obj();
  j.o["schema"] = Json::integer(1);
  j.o["machine"] = Json::str(report.machine);
  Json d = Json::obj();
  d.o["name"] = Json::str(report.dataset.name);
  d.o["samples"] = Json::integer(static_cast<long long>(report.dataset.samples));
  d.o["features"] = Json::integer(static_cast<long long>(report.dataset.features));
  d.o["classes"] = Json::integer(static_cast<long long>(report.dataset.classes));
  j.o["dataset"] = d;
  j.o["node_counts"] = sizes(report.node_counts);
  j.o["split_points"] = sizes(report.split_points);
  Json st = Json::arr();
  for (const TrialStats& s : report.stats) st.a.push_back(stats_json(s));
  j.o["stats"] = st;
  std::string out;
  write(j, 0, out);
  return out;
}

BenchmarkReport report_from_json(const std::string& text) {
  Parser ps{text};
  const Json j = ps.value();
  ps.ws();
  if (ps.p != text.size()) ps.bad("trailing characters");
  if (j.at("schema").kind != Json::Int || j.at("schema").i != 1)
    throw std::runtime_error("report_from_json: unsupported schema version");
  BenchmarkReport r;
  r.machine = j.at("machine").as_str();
  const Json& d = j.at("dataset");
  r.dataset.name = d.at("name").as_str();
  r.dataset.samples = d.at("samples").as_size();
  r.dataset.features = d.at("features").as_size();
  r.dataset.classes = d.at("classes").as_size();
  for (const Json& v : j.at("node_counts").a) r.node_counts.push_back(v.as_size());
  for (const Json& v : j.at("split_points").a) r.split_points.push_back(v.as_size());
  for (const Json& s : j.at("stats").a) r.stats.push_back(stats_from(s));
  return r;
}

void emit_report(const BenchmarkReport& report, const std::string& format, const std::string& path) {
  if (report.stats.empty()) throw std::invalid_argument("emit_report: empty report");
  if (format != "json" && format != "csv") throw std::invalid_argument("emit_report: unknown format '" + format + "'");
  std::ofstream out(path);
  if (!out) throw std::runtime_error("emit_report: cannot write " + path);
  if (format == "json") {
    out << report_to_json(report) << '\n';
  } else {
    out << "strategy,hidden_nodes,trials,mean_seconds,min_seconds,max_seconds,stddev_seconds,mean_solve_seconds,"
           "mean_accuracy\n";
    out.precision(17);
    for (const TrialStats& s : report.stats)
      out << s.strategy << ',' << s.hidden_nodes << ',' << s.trials << ',' << s.mean_seconds << ',' << s.min_seconds
          << ',' << s.max_seconds << ',' << s.stddev_seconds << ',' << s.mean_solve_seconds << ',' << s.mean_accuracy
          << '\n';
  }
  if (!out) throw std::runtime_error("emit_report: write failed for " + path);
}

std::vector<std::string> emit_plot_data(const BenchmarkReport& report, const std::string& path_prefix) {
  if (report.stats.empty()) throw std::invalid_argument("emit_plot_data: empty report");
  std::vector<std::string> order;
  for (const TrialStats& s : report.stats)
    if (std::find(order.begin(), order.end(), s.strategy) == order.end()) order.push_back(s.strategy);
  std::vector<std::string> paths;
  for (const std::string& strat : order) {
    std::string safe = strat;
    std::replace(safe.begin(), safe.end(), ':', '-');
    const std::string path = path_prefix + "." + safe + ".tsv";
    std::ofstream out(path);
    if (!out) throw std::runtime_error("emit_plot_data: cannot write " + path);
    out.precision(17);
    for (const TrialStats& s : report.stats)
      if (s.strategy == strat)
        out << s.hidden_nodes << '\t' << s.mean_seconds << '\t' << s.min_seconds << '\t' << s.max_seconds << '\n';
    if (!out) throw std::runtime_error("emit_plot_data: write failed for " + path);
    paths.push_back(path);
  }
  return paths;
}

}  // namespace rbpelm
