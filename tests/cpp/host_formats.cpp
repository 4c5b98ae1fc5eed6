// Host-only parts of the drop-in (no device work): the data layer (reference tests/test_data.cpp)
// and the benchmark report formats (tests/test_bench.cpp: JSON round trip, CSV / TSV emission),
// checked on hand-built reports.  Exit code 0 = all checks passed.
#include "rbpelm_b200.hpp"

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

using namespace rbpelm;

static int failures = 0;
#define CHECK(c)                                                 \
  do {                                                           \
    if (!(c)) {                                                  \
      std::printf("CHECK failed: %s (line %d)\n", #c, __LINE__); \
      ++failures;                                                \
    }                                                            \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f, const std::string& needle = "") {
  try {
    f();
  } catch (const E& e) {
    return needle.empty() || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

struct TempFile {
  std::string path;
  TempFile(const std::string& name, const std::string& text) : path("/tmp/rbpg_host_test_" + name) {
    std::ofstream(path) << text;
  }
  ~TempFile() { std::remove(path.c_str()); }
};

static TrialStats fake_stats(const std::string& strat, std::size_t nodes, double base) {
  TrialStats s;
  s.strategy = strat;
  s.hidden_nodes = nodes;
  s.trials = 2;
  for (int t = 0; t < 2; ++t) {
    TrialRecord r;
    r.seed = 40 + t;
    r.total_seconds = base * (1.0 + 0.1 * t) + 1e-17;
    r.solve_seconds = base / 3.0;
    r.hidden_seconds = base / 7.0;
    r.accuracy = 0.875 + t * 1e-3;
    r.rank = nodes - t;
    r.rank_known = true;
    r.ridge_applied = t == 1;
    r.fallback_to_direct = false;
    s.records.push_back(r);
  }
  s.mean_seconds = base * 1.05;
  s.min_seconds = base;
  s.max_seconds = base * 1.1;
  s.stddev_seconds = base * 0.0707106781186548;
  s.mean_solve_seconds = base / 3.0;
  s.mean_accuracy = 0.8755;
  return s;
}

int main() {
  // ---- load_csv (test_data.cpp:25-56)
  {
    TempFile f("basic.csv", "1.0,2.0,a\n3.0,4.0,b\n5.0,6.0,a\n");
    Dataset ds = load_csv(f.path);
    CHECK(ds.samples() == 3 && ds.features() == 2);
    CHECK((ds.class_names == std::vector<std::string>{"a", "b"}));
    CHECK(ds.y == DenseMatrix(3, 2, {1, 0, 0, 1, 1, 0}));
    CHECK(ds.x(2, 1) == 6.0);
  }
  {
    TempFile f("header.csv", "f1,label,f2\n1,x,2\n3,y,4\n");
    Dataset ds = load_csv(f.path, 1, true);
    CHECK(ds.samples() == 2 && ds.features() == 2);
    CHECK(ds.x == DenseMatrix(2, 2, {1, 2, 3, 4}));
    CHECK((ds.class_names == std::vector<std::string>{"x", "y"}));
  }
  {
    TempFile bad("bad.csv", "1,2,a\n1,oops,b\n");
    CHECK(throws<DataError>([&] { load_csv(bad.path); }, ":2"));
    TempFile ragged("ragged.csv", "1,2,a\n1,2,3,b\n");
    CHECK(throws<DataError>([&] { load_csv(ragged.path); }, "columns"));
    TempFile empty("empty.csv", "");
    CHECK(throws<DataError>([&] { load_csv(empty.path); }));
    CHECK(throws<DataError>([&] { load_csv("/nonexistent/file.csv"); }));
    TempFile inf("inf.csv", "1,inf,a\n");
    CHECK(throws<DataError>([&] { load_csv(inf.path); }, "non-numeric"));
    TempFile blank("blank.csv", "\n1,2,a\n\n3,4,b\n");
    CHECK(load_csv(blank.path).samples() == 2);
  }
  // ---- load_libsvm / save_libsvm (test_data.cpp:58-86)
  {
    TempFile f("basic.svm", "1 1:0.5 3:2.0\n2\n1 2:1.5\n");
    Dataset ds = load_libsvm(f.path);
    CHECK(ds.samples() == 3 && ds.features() == 3);
    CHECK(ds.x(0, 0) == 0.5 && ds.x(0, 1) == 0.0 && ds.x(0, 2) == 2.0);
    for (std::size_t j = 0; j < 3; ++j) CHECK(ds.x(1, j) == 0.0);
    CHECK((ds.class_names == std::vector<std::string>{"1", "2"}));
    TempFile b1("bad.svm", "1 1:0.5\n1 nonsense\n");
    CHECK(throws<DataError>([&] { load_libsvm(b1.path); }, ":2"));
    TempFile b2("bad0.svm", "1 0:0.5\n");
    CHECK(throws<DataError>([&] { load_libsvm(b2.path); }));
    Dataset s = synth(12, 5, 3, 77);
    const std::string path = "/tmp/rbpg_host_test_roundtrip.svm";
    save_libsvm(s, path);
    Dataset back = load_libsvm(path);
    std::remove(path.c_str());
    CHECK(back.x == s.x && back.y == s.y && back.class_names == s.class_names);
  }
  // ---- normalize (test_data.cpp:88-105)
  {
    Dataset raw;
    raw.x = DenseMatrix(3, 2, {0, 7, 5, 7, 10, 7});
    raw.y = DenseMatrix(3, 1, {1, 1, 1});
    raw.class_names = {"only"};
    Dataset ds = normalize(raw);
    CHECK(ds.x(0, 0) == -1.0 && ds.x(1, 0) == 0.0 && ds.x(2, 0) == 1.0);
    for (std::size_t i = 0; i < 3; ++i) CHECK(ds.x(i, 1) == 0.0);
    CHECK((ds.feature_ranges[0] == std::pair<double, double>{0.0, 10.0}));
    CHECK(normalize(ds).x == ds.x);
    CHECK(throws<DataError>([&] { normalize_with(raw, {{0.0, 1.0}}); }));
  }
  // ---- synth (test_data.cpp:107-128)
  {
    Dataset a = synth(30, 4, 3, 5), b = synth(30, 4, 3, 5);
    CHECK(a.x == b.x && a.y == b.y);
    CHECK(a.samples() == 30 && a.features() == 4 && a.classes() == 3);
    for (std::size_t i = 0; i < a.samples(); ++i) {
      double sum = 0.0;
      for (std::size_t j = 0; j < a.classes(); ++j) sum += a.y(i, j);
      CHECK(sum == 1.0);
      for (std::size_t j = 0; j < a.features(); ++j) CHECK(a.x(i, j) >= -1.0 && a.x(i, j) <= 1.0);
    }
    Dataset one = synth(5, 3, 1, 9);
    CHECK(one.classes() == 1);
    CHECK(throws<DataError>([&] { synth(0, 3, 1, 9); }));
  }
  // ---- report formats (test_bench.cpp:86-118), on a hand-built report
  {
    BenchmarkReport rep;
    rep.machine = "B200 \"sm_100a\"\tx";
    rep.dataset = {"synth", 60, 5, 2};
    rep.node_counts = {6, 10};
    rep.split_points = {3, 5};
    rep.stats = {fake_stats("direct", 6, 0.5), fake_stats("rank", 6, 0.25), fake_stats("direct", 10, 1.5),
                 fake_stats("rank:1e-06", 10, 0.3)};
    const std::string text = report_to_json(rep);
    BenchmarkReport back = report_from_json(text);
    CHECK(report_to_json(back) == text);
    CHECK(back.stats.size() == 4 && back.machine == rep.machine);
    CHECK(back.stats[1].records[0].total_seconds == rep.stats[1].records[0].total_seconds);
    CHECK(back.stats[3].records[1].ridge_applied && back.stats[3].records[1].rank == 9);
    CHECK(text.find("\"schema\": 1") != std::string::npos);
    CHECK(throws<std::runtime_error>([&] { report_from_json("{\"schema\": 2}"); }, "schema"));
    CHECK(throws<std::runtime_error>([&] { report_from_json("{\"schema\": 1"); }));

    const std::string csv = "/tmp/rbpg_host_test_report.csv";
    emit_report(rep, "csv", csv);
    std::ifstream in(csv);
    std::string line;
    std::size_t lines = 0;
    while (std::getline(in, line)) ++lines;
    std::remove(csv.c_str());
    CHECK(lines == rep.stats.size() + 1);
    const std::string js = "/tmp/rbpg_host_test_report.json";
    emit_report(rep, "json", js);
    std::stringstream buf;
    buf << std::ifstream(js).rdbuf();
    std::remove(js.c_str());
    CHECK(report_from_json(buf.str()).stats.size() == 4);

    auto paths = emit_plot_data(rep, "/tmp/rbpg_host_test_plot");
    CHECK(paths.size() == 3);  // direct, rank, rank:1e-06 -> rank-1e-06
    CHECK(paths[2].find("rank-1e-06.tsv") != std::string::npos);
    for (const auto& p : paths) {
      std::ifstream pin(p);
      std::string row;
      while (std::getline(pin, row)) {
        std::size_t fields = 1;
        for (char ch : row) fields += ch == '\t';
        CHECK(fields == 4);
      }
      std::remove(p.c_str());
    }
    CHECK(throws<std::invalid_argument>([&] { emit_report(rep, "xml", "/tmp/x"); }));
    CHECK(throws<std::runtime_error>([&] { emit_report(rep, "json", "/nonexistent_dir/x.json"); }));
    CHECK(throws<std::invalid_argument>([&] { emit_report(BenchmarkReport{}, "json", "/tmp/x"); }));
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
