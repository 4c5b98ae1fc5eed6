// The reference's trial / sweep protocol (tests/test_bench.cpp:18-84) run through the device
// train().  Exit code 0 = all checks passed.
#include "rbpelm_b200.hpp"

#include <cstdio>
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

static ElmParams small_params(const Dataset& ds, std::size_t nodes, std::uint64_t seed = 0) {
  return ElmParams{ds.features(), nodes, ds.classes(), Activation::Sigmoid, seed};
}

int main() {
  {  // single trial collapses min, mean and max
    Dataset ds = synth(40, 5, 2, 1);
    TrialStats s = run_trials(ds, small_params(ds, 8), SolverStrategy::rank_based(), 1);
    CHECK(s.trials == 1 && s.min_seconds == s.mean_seconds && s.max_seconds == s.mean_seconds);
    CHECK(s.stddev_seconds == 0.0);
  }
  {  // same base seed reproduces the accuracies, per-trial reseeding from the base
    Dataset ds = synth(50, 6, 3, 2);
    TrialStats a = run_trials(ds, small_params(ds, 10, 4), SolverStrategy::direct(), 3);
    TrialStats b = run_trials(ds, small_params(ds, 10, 4), SolverStrategy::direct(), 3);
    CHECK(a.records.size() == b.records.size());
    for (std::size_t i = 0; i < a.records.size(); ++i) {
      CHECK(a.records[i].accuracy == b.records[i].accuracy);
      CHECK(a.records[i].seed == 4 + i);
    }
  }
  {  // ordered statistics; df and rank give the same accuracies (the paper's Table-2 phenomenon)
    Dataset ds = synth(60, 8, 2, 3);
    TrialStats df = run_trials(ds, small_params(ds, 12), SolverStrategy::df_split(6), 4);
    TrialStats rb = run_trials(ds, small_params(ds, 12), SolverStrategy::rank_based(), 4);
    for (const TrialStats* s : {&df, &rb})
      CHECK(s->min_seconds <= s->mean_seconds && s->mean_seconds <= s->max_seconds && s->stddev_seconds >= 0.0);
    for (std::size_t i = 0; i < 4; ++i) CHECK(df.records[i].accuracy == rb.records[i].accuracy);
  }
  {  // df split sweep
    Dataset ds = synth(50, 5, 2, 4);
    ElmParams p = small_params(ds, 12);
    CHECK(sweep_df_splits(ds, p, {6}, 2).stats.size() == 1);
    SweepResult sw = sweep_df_splits(ds, p, {3, 6, 9}, 2);
    CHECK(sw.stats.size() == 3);
    CHECK(sw.stats[sw.worst_index].mean_seconds >= sw.stats[sw.best_index].mean_seconds);
    CHECK(sw.stats[0].mean_accuracy == sw.stats[2].mean_accuracy);  // symmetric splits
    bool threw = false;
    try { sweep_df_splits(ds, p, {12}, 2); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { sweep_df_splits(ds, p, {}, 2); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
  }
  {  // node sweep cross product, JSON round trip of a measured report
    Dataset ds = synth(60, 5, 2, 5);
    std::vector<SolverStrategy> st{SolverStrategy::direct(), SolverStrategy::rank_based()};
    BenchmarkReport rep = sweep_nodes(ds, small_params(ds, 0), {8, 12, 16}, st, 2, "test-machine", "synth");
    CHECK(rep.stats.size() == 6 && rep.dataset.samples == 60);
    CHECK(sweep_nodes(ds, small_params(ds, 0), {8}, {SolverStrategy::direct()}, 1).stats.size() == 1);
    bool threw = false;
    try { sweep_nodes(ds, small_params(ds, 0), {100}, st, 1); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    rep.split_points = {3, 5};
    const std::string text = report_to_json(rep);
    CHECK(report_to_json(report_from_json(text)) == text);
    CHECK(report_from_json(text).stats[1].records[0].total_seconds == rep.stats[1].records[0].total_seconds);
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
