// Host-side Q1 assembly into 9-diagonal coefficient arrays.
//
// Restates the reference's element formulas (fem.cpp:35-106: 2x2 Gauss mass,
// stiffness and SUPG convection-diffusion elements) and its Dirichlet
// elimination (fem.cpp:109-140), but assembles straight into the
// structure-of-arrays 9-point layout the device kernels read (Op9) instead
// of a triplet buffer + CSR. Entry d = (dy+1)*3+(dx+1) for node i holds
// A(i, i + dx + dy*nx); neighbours outside the interior hold 0.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

namespace ocb {

inline int level_nx(int level) { return (1 << level) - 1; }
inline long long level_n(int level)
{
    const long long nx = level_nx(level);
    return nx * nx;
}

enum class AssembleKind { mass = 0, poisson = 1, convdiff = 2, partial_mass = 3, lumped = 4 };

std::vector<double> assemble_mass9(int level);
std::vector<double> assemble_poisson9(int level);
std::vector<double> assemble_convdiff9(int level, double eps, bool supg = true);
std::vector<double> assemble_partial_mass9(int level, const double obs[4]);
/// Row sums of the Dirichlet-eliminated consistent mass (qp.cpp:137).
std::vector<double> lumped_diag(int level);
/// Transpose of a 9-point operator: T(i, i+d) = A(i+d, i).
std::vector<double> transpose9(const std::vector<double>& coef, int level);
/// The grid-constant stencils without assembling the level: the mass matrix
/// scales exactly with h^2 (a power of 4) and the Q1 Poisson stiffness is
/// h-independent in 2D, so the centre row of the level-3 assembly, scaled by
/// 4^(3 - level), is bitwise the centre row of the full assembly
/// (tests/test_assembly_shortcut.py). what: 0 mass, 1 Poisson.
void stencil9(int what, int level, double c[9]);
/// lumped_diag from the constant mass stencil: row sums over the in-domain
/// neighbours in ascending column order (bitwise lumped_diag).
std::vector<double> lumped_from_stencil(const double cM[9], int level);
/// y = M f with the constant mass stencil, dropped boundary neighbours.
std::vector<double> apply_stencil(const double c[9], int level, const std::vector<double>& f);

} // namespace ocb
