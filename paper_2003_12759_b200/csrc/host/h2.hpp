// Small dense second-order / H2 helpers for the AIRGA driver
// (proj/src/h2.cpp:11-79, proj/src/airga.cpp:319-384). Host, O(r^3).
#pragma once

#include <vector>

#include "small_dense.hpp"

namespace mpg::host {

struct StateSpace {
  Mat a, b, c;  // ns x ns, ns x m, q x ns
};
// Companion form of m x'' + d x' + k x = f u, y = c^T x (h2.cpp:11-26).
StateSpace second_order_to_state_space(const Mat& m, const Mat& d, const Mat& k, const Mat& f, const Mat& c);
// H2 norm through the diagonalised Lyapunov solve (h2.cpp:28-60); +inf when A
// is not asymptotically stable or its eigenvectors are not independent.
double h2_norm(const StateSpace& sys);
double h2_distance(const StateSpace& a, const StateSpace& b);
// update_expansion_points (airga.cpp:319-384).
std::vector<double> update_expansion_points(const Mat& m, const Mat& d, const Mat& k,
                                            const std::vector<double>& current);

}  // namespace mpg::host
