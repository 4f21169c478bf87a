// fb_host.h -- host-side precompute and input synthesis for the B200 engine.
//
//  * analytic tensor K (the form-dependent, mesh-independent reference tensor
//    built once on the host and uploaded into the kernel's constant bank),
//    following reference src/forms.cpp:63-246 + src/reference.cpp:39-138;
//  * the reference's structured / jittered simplicial mesh generators
//    (src/geometry.cpp:164-262), reproduced bit for bit so benchmark and test
//    inputs are the reference's inputs without the reference present;
//  * a host Jacobian / geometry tensor for the C++ API's element_jacobian.
// Errors are thrown as the reference's exception types and texts.
#pragma once

#include <cstdint>
#include <vector>

namespace fbh {

int krows(int op, int dim);
int ncoef(int op, int dim);
int64_t k_len(int op, int dim);
void check_dim(int dim);  // throws std::invalid_argument

// K in the reference AnalyticTensor layout
//   ((i + j*krows)*ncoef + c)*dim^2 + mu*dim + nu.
std::vector<double> build_analytic_tensor(int op, int dim);

// Quadrature rule of degree 1..3 on the reference simplex (points row-major).
void quadrature(int dim, int degree, std::vector<double>& points, std::vector<double>& weights);

void structured_mesh_sizes(int dim, int n, int64_t& nv, int64_t& ne);
void structured_mesh(int dim, int n, double* vertices, int32_t* cells);
void jitter_mesh(int dim, double* vertices, int64_t nv, const int32_t* cells, int64_t ne,
                 double magnitude, uint64_t seed);

// src/geometry.cpp:27-66 / :286-302 (host, FP64).  Returns false if det <= 0.
bool jacobian(int dim, const double* x, double* j, double* jinv, double* det);
void geometry_tensor(int dim, const double* jinv, double det, double* g);
// Throws std::runtime_error("degenerate element: det(J) <= 0 in cell N").
void check_cells(int dim, const double* vertices, int64_t nv, const int32_t* cells, int64_t ne);

}  // namespace fbh
