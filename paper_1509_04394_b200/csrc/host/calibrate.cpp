// Cost-model calibration (fp_calibrate_csv): the reference's least-squares
// fit of the planner's four cost parameters to measured kernel times
// (proj/src/calibrate.cpp:10-101).  The features and the CSV format are the
// reference's; the solve restates Eigen's ColPivHouseholderQR (Householder QR
// with column pivoting, rank threshold eps * min(rows, cols) relative to the
// largest pivot), so the fitted parameters agree with the reference to
// rounding, not bit for bit (Eigen is not available in this image).
#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/fuseplan/fuseplan.hpp"

namespace fuseplan {

struct Measurement {
  int n_kernels = 1;
  std::int64_t blocks = 1;
  TileShape tile;
  Halo halo;
  double measured_time = 0.0;
};

// calibrate.cpp:10-24
std::array<double, 4> cost_features(const Measurement& m) {
  require(m.n_kernels >= 1 && m.blocks >= 1, ErrorKind::Input,
          "measurement counts must be >= 1");
  const double out_elems = double(m.blocks) * double(m.tile.volume());
  const double in_elems = double(m.blocks) * double(input_box(m.tile, m.halo).volume());
  const double window = double(m.halo.dx() + 1) * (m.halo.dy() + 1) * (m.halo.dt() + 1);
  return {in_elems + out_elems, m.n_kernels * out_elems * (window + 1.0),
          m.n_kernels * out_elems, 1.0};
}

// calibrate.cpp:56-99
std::vector<Measurement> parse_measurements_csv(const std::string& text) {
  std::vector<Measurement> rows;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    if (lineno == 1 && line.find("n_kernels") != std::string::npos) continue;
    std::istringstream ls(line);
    std::vector<double> fields;
    std::string cell;
    while (std::getline(ls, cell, ',')) {
      try {
        fields.push_back(std::stod(cell));
      } catch (const std::exception&) {
        throw Error(ErrorKind::Input, "measurements line " + std::to_string(lineno) +
                                          ": bad number '" + cell + "'");
      }
    }
    require(fields.size() == 12, ErrorKind::Input,
            "measurements line " + std::to_string(lineno) + ": expected 12 columns, got " +
                std::to_string(fields.size()));
    Measurement m;
    m.n_kernels = int(fields[0]);
    m.blocks = std::int64_t(fields[1]);
    m.tile = TileShape{int(fields[2]), int(fields[3]), int(fields[4])};
    m.halo = Halo{int(fields[5]), int(fields[6]), int(fields[7]),
                  int(fields[8]), int(fields[9]), int(fields[10])};
    m.measured_time = fields[11];
    m.halo.validate();
    require(m.tile.x >= 1 && m.tile.y >= 1 && m.tile.t >= 1, ErrorKind::Input,
            "measurements line " + std::to_string(lineno) + ": tile dims must be >= 1");
    rows.push_back(m);
  }
  require(!rows.empty(), ErrorKind::Input, "no measurement rows");
  return rows;
}

// Least squares min |A x - y| (A: n x 4, row-major) by Householder QR with
// column pivoting; returns the rank and x (valid when rank == 4).
int lstsq_colpiv(std::vector<double> a, std::vector<double> y, int n, double x[4]) {
  constexpr int P = 4;
  int perm[P] = {0, 1, 2, 3};
  std::vector<double> norms(P);
  for (int j = 0; j < P; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i * P + j] * a[i * P + j];
    norms[j] = s;
  }
  const int steps = std::min(n, P);
  double maxpivot = 0.0;
  std::vector<double> diag(P, 0.0);
  for (int k = 0; k < steps; ++k) {
    // pivot: the remaining column of largest norm
    int best = k;
    for (int j = k + 1; j < P; ++j)
      if (norms[j] > norms[best]) best = j;
    if (best != k) {
      for (int i = 0; i < n; ++i) std::swap(a[i * P + k], a[i * P + best]);
      std::swap(norms[k], norms[best]);
      std::swap(perm[k], perm[best]);
    }
    // Householder vector for column k, rows k..n-1
    double alpha = 0.0;
    for (int i = k; i < n; ++i) alpha += a[i * P + k] * a[i * P + k];
    alpha = std::sqrt(alpha);
    if (a[k * P + k] > 0) alpha = -alpha;
    const double v0 = a[k * P + k] - alpha;
    double vnorm2 = v0 * v0;
    for (int i = k + 1; i < n; ++i) vnorm2 += a[i * P + k] * a[i * P + k];
    diag[k] = alpha;
    maxpivot = std::max(maxpivot, std::fabs(alpha));
    if (vnorm2 > 0.0) {
      auto vi = [&](int i) { return i == k ? v0 : a[i * P + k]; };
      for (int j = k + 1; j < P; ++j) {
        double d = 0.0;
        for (int i = k; i < n; ++i) d += vi(i) * a[i * P + j];
        const double f = 2.0 * d / vnorm2;
        for (int i = k; i < n; ++i) a[i * P + j] -= f * vi(i);
      }
      double d = 0.0;
      for (int i = k; i < n; ++i) d += vi(i) * y[i];
      const double f = 2.0 * d / vnorm2;
      for (int i = k; i < n; ++i) y[i] -= f * vi(i);
    }
    a[k * P + k] = alpha;
    // downdate the remaining column norms
    for (int j = k + 1; j < P; ++j) {
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += a[i * P + j] * a[i * P + j];
      norms[j] = s;
    }
  }
  const double thresh = std::numeric_limits<double>::epsilon() * double(steps);
  int rank = 0;
  for (int k = 0; k < steps; ++k)
    if (std::fabs(diag[k]) > thresh * maxpivot) ++rank;
  if (rank < P) return rank;
  double z[P];
  for (int k = P - 1; k >= 0; --k) {
    double s = y[k];
    for (int j = k + 1; j < P; ++j) s -= a[k * P + j] * z[j];
    z[k] = s / a[k * P + k];
  }
  for (int k = 0; k < P; ++k) x[perm[k]] = z[k];
  return rank;
}

// calibrate.cpp:31-54
void calibrate_rows(const std::vector<Measurement>& rows, double params[4], double* rms) {
  require(rows.size() >= 4, ErrorKind::Input, "calibration needs >= 4 measurements");
  const int n = int(rows.size());
  std::vector<double> a(std::size_t(n) * 4), y(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    const auto f = cost_features(rows[std::size_t(i)]);
    for (int j = 0; j < 4; ++j) a[std::size_t(i) * 4 + j] = f[std::size_t(j)];
    y[std::size_t(i)] = rows[std::size_t(i)].measured_time;
  }
  const int rank = lstsq_colpiv(a, y, n, params);
  require(rank == 4, ErrorKind::Input,
          "calibration design matrix is rank deficient; vary tile, halo and kernel counts "
          "across measurements");
  double sq = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = -y[std::size_t(i)];
    for (int j = 0; j < 4; ++j) r += a[std::size_t(i) * 4 + j] * params[j];
    sq += r * r;
  }
  *rms = std::sqrt(sq / double(n));
}

void calibrate_csv(const std::string& text, double params[4], double* rms) {
  calibrate_rows(parse_measurements_csv(text), params, rms);
}

}  // namespace fuseplan
