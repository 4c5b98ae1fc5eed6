// Host-side dataset formats feeding train() -- the reference's data layer (proj/src/data.cpp,
// include/rbpelm/data.hpp).  Behaviour restated from the reference:
//   * load_csv (data.cpp:64-117): blank lines skipped, optional header, label column (last by
//     default), every row the width of the first, numeric cells finite, classes one-hot in
//     first-appearance order; DataError messages carry "path:line" and the column.
//   * load_libsvm (data.cpp:119-176): "label idx:val ..." with 1-based indices, width = largest
//     index (>= 1), malformed tokens reported with the line number.
//   * save_libsvm (data.cpp:178-193): label = arg-max of the one-hot row, non-zero entries only,
//     17 significant digits (exact round trip).
//   * normalize / normalize_with (data.cpp:195-227): per-feature min-max onto [-1, 1], constant
//     features to 0, values clamped, ranges recorded.
//   * synth (data.cpp:229-253): one Gaussian cluster per class, centres U(-1, 1), noise N(0, 0.4),
//     row i in class i % classes, drawn from std::mt19937_64(seed) through the standard library
//     distributions (the same libstdc++ draws as the reference build), then normalized.
#include "../../include/rbpelm_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>

namespace rbpelm {

namespace {

std::string strip(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

// comma cells; a trailing separator yields a trailing empty cell
std::vector<std::string> cells_of(const std::string& line) {
  std::vector<std::string> out;
  std::size_t start = 0;
  while (true) {
    const auto comma = line.find(',', start);
    if (comma == std::string::npos) {
      if (start < line.size() || (!line.empty() && line.back() == ',')) out.push_back(line.substr(start));
      break;
    }
    out.push_back(line.substr(start, comma - start));
    start = comma + 1;
  }
  if (line.empty()) out.clear();
  return out;
}

bool to_finite(const std::string& token, double& v) {
  const std::string t = strip(token);
  if (t.empty()) return false;
  char* end = nullptr;
  v = std::strtod(t.c_str(), &end);
  return end == t.c_str() + t.size() && std::isfinite(v);
}

std::size_t class_id(std::vector<std::string>& names, const std::string& label) {
  for (std::size_t i = 0; i < names.size(); ++i)
    if (names[i] == label) return i;
  names.push_back(label);
  return names.size() - 1;
}

Dataset one_hot(std::size_t rows, std::size_t feats, const std::vector<double>& x,
                const std::vector<std::size_t>& labels, std::vector<std::string> names) {
  Dataset ds;
  ds.x = DenseMatrix(rows, feats, std::vector<double>(x));
  ds.y = DenseMatrix(rows, names.size(), 0.0);
  for (std::size_t i = 0; i < rows; ++i) ds.y(i, labels[i]) = 1.0;
  ds.class_names = std::move(names);
  return ds;
}

}  // namespace

Dataset load_csv(const std::string& path, int label_column, bool has_header) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open " + path);
  std::vector<double> values;
  std::vector<std::size_t> labels;
  std::vector<std::string> names;
  std::size_t width = 0, lineno = 0;
  std::string line;
  while (std::getline(in, line)) {
    ++lineno;
    if (has_header && lineno == 1) continue;
    if (strip(line).empty()) continue;
    const std::vector<std::string> cells = cells_of(line);
    if (width == 0) {
      width = cells.size();
      if (width < 2)
        throw DataError(path + ":" + std::to_string(lineno) + ": need at least one feature and one label column");
    } else if (cells.size() != width) {
      throw DataError(path + ":" + std::to_string(lineno) + ": expected " + std::to_string(width) +
                      " columns, got " + std::to_string(cells.size()));
    }
    const std::size_t lab = label_column < 0 ? width - 1 : static_cast<std::size_t>(label_column);
    if (lab >= width)
      throw DataError(path + ": label column " + std::to_string(lab) + " out of range for " + std::to_string(width) +
                      " columns");
    for (std::size_t c = 0; c < width; ++c) {
      if (c == lab) continue;
      double v = 0.0;
      if (!to_finite(cells[c], v))
        throw DataError(path + ":" + std::to_string(lineno) + ": column " + std::to_string(c + 1) +
                        ": non-numeric cell '" + strip(cells[c]) + "'");
      values.push_back(v);
    }
    labels.push_back(class_id(names, strip(cells[lab])));
  }
  if (labels.empty()) throw DataError(path + ": no data rows");
  return one_hot(labels.size(), width - 1, values, labels, std::move(names));
}

Dataset load_libsvm(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open " + path);
  std::vector<std::vector<std::pair<std::size_t, double>>> rows;
  std::vector<std::size_t> labels;
  std::vector<std::string> names;
  std::size_t width = 0, lineno = 0;
  std::string line;
  while (std::getline(in, line)) {
    ++lineno;
    const std::string t = strip(line);
    if (t.empty()) continue;
    std::istringstream is(t);
    std::string label, tok;
    is >> label;
    labels.push_back(class_id(names, label));
    std::vector<std::pair<std::size_t, double>> entries;
    while (is >> tok) {
      const auto colon = tok.find(':');
      bool ok = colon != std::string::npos && colon > 0;
      long idx = 0;
      double v = 0.0;
      if (ok) {
        char* end = nullptr;
        const std::string head = tok.substr(0, colon);
        idx = std::strtol(head.c_str(), &end, 10);
        ok = end == head.c_str() + head.size() && idx >= 1;
      }
      if (ok) ok = to_finite(tok.substr(colon + 1), v);
      if (!ok) throw DataError(path + ":" + std::to_string(lineno) + ": malformed index:value token '" + tok + "'");
      width = std::max(width, static_cast<std::size_t>(idx));
      entries.emplace_back(static_cast<std::size_t>(idx) - 1, v);
    }
    rows.push_back(std::move(entries));
  }
  if (rows.empty()) throw DataError(path + ": no data rows");
  if (width == 0) width = 1;  // rows without features still give one (zero) column
  std::vector<double> dense(rows.size() * width, 0.0);
  for (std::size_t i = 0; i < rows.size(); ++i)
    for (const auto& e : rows[i]) dense[i * width + e.first] = e.second;
  return one_hot(rows.size(), width, dense, labels, std::move(names));
}

void save_libsvm(const Dataset& ds, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write " + path);
  out.precision(17);
  for (std::size_t i = 0; i < ds.samples(); ++i) {
    std::size_t lab = 0;
    for (std::size_t j = 1; j < ds.classes(); ++j)
      if (ds.y(i, j) > ds.y(i, lab)) lab = j;
    out << ds.class_names[lab];
    for (std::size_t j = 0; j < ds.features(); ++j)
      if (ds.x(i, j) != 0.0) out << ' ' << (j + 1) << ':' << ds.x(i, j);
    out << '\n';
  }
  if (!out) throw DataError("write failed for " + path);
}

Dataset normalize_with(const Dataset& ds, const std::vector<std::pair<double, double>>& ranges) {
  if (ranges.size() != ds.features())
    throw DataError("normalize: " + std::to_string(ranges.size()) + " ranges for " + std::to_string(ds.features()) +
                    " features");
  Dataset out = ds;
  for (std::size_t j = 0; j < ds.features(); ++j) {
    const double lo = ranges[j].first, span = ranges[j].second - ranges[j].first;
    for (std::size_t i = 0; i < ds.samples(); ++i) {
      const double v = span > 0.0 ? 2.0 * (ds.x(i, j) - lo) / span - 1.0 : 0.0;
      out.x(i, j) = std::min(1.0, std::max(-1.0, v));
    }
  }
  out.feature_ranges = ranges;
  return out;
}

Dataset normalize(const Dataset& ds) {
  std::vector<std::pair<double, double>> ranges(ds.features());
  for (std::size_t j = 0; j < ds.features(); ++j) {
    double lo = ds.x(0, j), hi = ds.x(0, j);
    for (std::size_t i = 1; i < ds.samples(); ++i) {
      lo = std::min(lo, ds.x(i, j));
      hi = std::max(hi, ds.x(i, j));
    }
    ranges[j] = {lo, hi};
  }
  return normalize_with(ds, ranges);
}

Dataset synth(std::size_t samples, std::size_t features, std::size_t classes, std::uint64_t seed) {
  if (samples < 1 || features < 1 || classes < 1) throw DataError("synth: samples, features and classes must be >= 1");
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> centre(-1.0, 1.0);
  std::normal_distribution<double> noise(0.0, 0.4);
  std::vector<double> mu(classes * features);
  for (double& v : mu) v = centre(gen);  // class-major, feature-minor
  Dataset ds;
  ds.x = DenseMatrix(samples, features, 0.0);
  ds.y = DenseMatrix(samples, classes, 0.0);
  for (std::size_t i = 0; i < samples; ++i) {
    const std::size_t c = i % classes;
    for (std::size_t j = 0; j < features; ++j) ds.x(i, j) = mu[c * features + j] + noise(gen);
    ds.y(i, c) = 1.0;
  }
  for (std::size_t c = 0; c < classes; ++c) ds.class_names.push_back("c" + std::to_string(c));
  return normalize(ds);
}

}  // namespace rbpelm
