// Host-side Q1 assembly into 9-diagonal coefficient arrays (see assembly.hpp).
#include "assembly.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace ocb {

namespace {

// 2x2 Gauss points on [-1,1]^2 (fem.cpp:16-19), corner order SW, SE, NE, NW.
constexpr double kG = 0.57735026918962576;
constexpr double kQ[4][2] = {{-kG, -kG}, {kG, -kG}, {kG, kG}, {-kG, kG}};

using Elem = std::array<std::array<double, 4>, 4>;

void shape(double xi, double eta, double N[4])
{
    N[0] = 0.25 * (1 - xi) * (1 - eta);
    N[1] = 0.25 * (1 + xi) * (1 - eta);
    N[2] = 0.25 * (1 + xi) * (1 + eta);
    N[3] = 0.25 * (1 - xi) * (1 + eta);
}

void shape_grad(double xi, double eta, double G[4][2])
{
    G[0][0] = -0.25 * (1 - eta); G[0][1] = -0.25 * (1 - xi);
    G[1][0] = 0.25 * (1 - eta);  G[1][1] = -0.25 * (1 + xi);
    G[2][0] = 0.25 * (1 + eta);  G[2][1] = 0.25 * (1 + xi);
    G[3][0] = -0.25 * (1 + eta); G[3][1] = 0.25 * (1 - xi);
}

// fem.cpp:35-45
Elem element_mass(double h)
{
    Elem m{};
    const double detj = h * h / 4.0;
    for (const auto& q : kQ) {
        double N[4];
        shape(q[0], q[1], N);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) m[i][j] += N[i] * N[j] * detj;
    }
    return m;
}

// fem.cpp:47-59
Elem element_stiffness(double h)
{
    Elem k{};
    const double detj = h * h / 4.0;
    const double s = 2.0 / h;
    for (const auto& q : kQ) {
        double G[4][2];
        shape_grad(q[0], q[1], G);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                k[i][j] += s * s * (G[i][0] * G[j][0] + G[i][1] * G[j][1]) * detj;
    }
    return k;
}

// default_wind (fem.cpp:164-169)
void wind(double x1, double x2, double w[2])
{
    w[0] = 2.0 * x2 * (1.0 - x1 * x1);
    w[1] = -2.0 * x1 * (1.0 - x2 * x2);
}

double delta_for(double h, double eps, double x0, double y0, bool supg)
{
    double wc[2];
    wind(x0 + 0.5 * h, y0 + 0.5 * h, wc);
    const double wnorm = std::hypot(wc[0], wc[1]);
    double delta = 0.0;
    if (supg && wnorm > 1e-14) {
        const double peclet = wnorm * h / (2.0 * eps);
        delta = h / (2.0 * wnorm) * std::max(0.0, 1.0 - 1.0 / peclet);
    }
    return delta;
}

// fem.cpp:61-106
Elem element_convdiff(double h, int ex, int ey, double eps, bool supg)
{
    const double x0 = ex * h, y0 = ey * h;
    const double detj = h * h / 4.0;
    const double s = 2.0 / h;
    Elem a = element_stiffness(h);
    for (auto& row : a)
        for (auto& v : row) v *= eps;
    const double delta = delta_for(h, eps, x0, y0, supg);
    for (const auto& q : kQ) {
        double N[4], G[4][2], w[2];
        shape(q[0], q[1], N);
        shape_grad(q[0], q[1], G);
        const double xq = x0 + 0.5 * h * (q[0] + 1.0);
        const double yq = y0 + 0.5 * h * (q[1] + 1.0);
        wind(xq, yq, w);
        double wg[4];
        for (int i = 0; i < 4; ++i) wg[i] = s * (w[0] * G[i][0] + w[1] * G[i][1]);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                a[i][j] += wg[j] * N[i] * detj;
                if (delta > 0.0) a[i][j] += delta * wg[j] * wg[i] * detj;
            }
    }
    return a;
}

// Scatter element matrices into the 9-diagonal arrays in element order
// (ey, ex ascending), dropping Dirichlet vertices (fem.cpp:118-140).
template <typename ElemFn>
std::vector<double> assemble(int level, ElemFn&& element)
{
    const int nx = level_nx(level);
    const int ne = 1 << level;
    const long long n = (long long)nx * nx;
    std::vector<double> coef(9 * static_cast<std::size_t>(n), 0.0);
    static const int lx[4] = {0, 1, 1, 0}, ly[4] = {0, 0, 1, 1};
    for (int ey = 0; ey < ne; ++ey)
        for (int ex = 0; ex < ne; ++ex) {
            const Elem a = element(ex, ey);
            for (int i = 0; i < 4; ++i) {
                const int gxi = ex + lx[i], gyi = ey + ly[i];
                if (gxi < 1 || gxi > nx || gyi < 1 || gyi > nx) continue;
                const long long row = (long long)(gyi - 1) * nx + (gxi - 1);
                for (int j = 0; j < 4; ++j) {
                    const int gxj = ex + lx[j], gyj = ey + ly[j];
                    if (gxj < 1 || gxj > nx || gyj < 1 || gyj > nx) continue;
                    const int d = (gyj - gyi + 1) * 3 + (gxj - gxi + 1);
                    coef[static_cast<std::size_t>(d * n + row)] += a[i][j];
                }
            }
        }
    return coef;
}

void check_level(int level)
{
    if (level < 1 || level > 14) throw std::invalid_argument("Grid: level out of range");
}

} // namespace

std::vector<double> assemble_mass9(int level)
{
    check_level(level);
    const Elem m = element_mass(1.0 / double(1 << level));
    return assemble(level, [&](int, int) { return m; });
}

std::vector<double> assemble_poisson9(int level)
{
    check_level(level);
    const Elem k = element_stiffness(1.0 / double(1 << level));
    return assemble(level, [&](int, int) { return k; });
}

std::vector<double> assemble_convdiff9(int level, double eps, bool supg)
{
    check_level(level);
    if (eps <= 0.0) throw std::invalid_argument("assemble_convdiff: eps must be positive");
    const double h = 1.0 / double(1 << level);
    return assemble(level, [&](int ex, int ey) { return element_convdiff(h, ex, ey, eps, supg); });
}

std::vector<double> assemble_partial_mass9(int level, const double obs[4])
{
    check_level(level);
    const double h = 1.0 / double(1 << level);
    const Elem m = element_mass(h);
    const Elem zero{};
    const double tol = 1e-12; // ObservationRegion::contains_box (grid.hpp:53-57)
    return assemble(level, [&](int ex, int ey) {
        const double x0 = ex * h, x1 = (ex + 1) * h, y0 = ey * h, y1 = (ey + 1) * h;
        const bool in = x0 >= obs[0] - tol && x1 <= obs[1] + tol && y0 >= obs[2] - tol &&
                        y1 <= obs[3] + tol;
        return in ? m : zero;
    });
}

std::vector<double> lumped_diag(int level)
{
    const std::vector<double> m = assemble_mass9(level);
    const long long n = level_n(level);
    std::vector<double> d(static_cast<std::size_t>(n), 0.0);
    // row_sums in ascending column order (sparse.cpp row_sums)
    for (long long i = 0; i < n; ++i)
        for (int k = 0; k < 9; ++k) d[i] += m[k * n + i];
    return d;
}

std::vector<double> transpose9(const std::vector<double>& coef, int level)
{
    const int nx = level_nx(level);
    const long long n = (long long)nx * nx;
    std::vector<double> t(coef.size(), 0.0);
    for (int gy = 0; gy < nx; ++gy)
        for (int gx = 0; gx < nx; ++gx) {
            const long long i = (long long)gy * nx + gx;
            // T(i, i+off(e)) = A(j, i) with j = i+off(e), i.e. entry 8-e of row j
            for (int e = 0; e < 9; ++e) {
                const int jx = gx + e % 3 - 1, jy = gy + e / 3 - 1;
                if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
                const long long j = (long long)jy * nx + jx;
                t[e * n + i] = coef[(8 - e) * n + j];
            }
        }
    return t;
}

void stencil9(int what, int level, double c[9])
{
    constexpr int L0 = 3;
    const std::vector<double> a = what == 0 ? assemble_mass9(L0) : assemble_poisson9(L0);
    const int nx = level_nx(L0);
    const long long n = (long long)nx * nx, mid = (long long)(nx / 2) * nx + nx / 2;
    double scale = 1.0;
    if (what == 0)
        for (int l = L0; l < level; ++l) scale *= 0.25; // exact: powers of two
    for (int d = 0; d < 9; ++d) c[d] = what == 0 ? a[d * n + mid] * scale : a[d * n + mid];
    if (what == 0 && level < L0) { // coarser than the reference grid: scale up
        double up = 1.0;
        for (int l = level; l < L0; ++l) up *= 4.0;
        for (int d = 0; d < 9; ++d) c[d] = a[d * n + mid] * up;
    }
}

std::vector<double> lumped_from_stencil(const double cM[9], int level)
{
    const int nx = level_nx(level);
    std::vector<double> out((std::size_t)nx * nx, 0.0);
    for (int gy = 0; gy < nx; ++gy)
        for (int gx = 0; gx < nx; ++gx) {
            double s = 0.0;
            for (int d = 0; d < 9; ++d) {
                const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
                s += cM[d];
            }
            out[(std::size_t)gy * nx + gx] = s;
        }
    return out;
}

std::vector<double> apply_stencil(const double c[9], int level, const std::vector<double>& f)
{
    const int nx = level_nx(level);
    std::vector<double> out((std::size_t)nx * nx, 0.0);
    for (int gy = 0; gy < nx; ++gy)
        for (int gx = 0; gx < nx; ++gx) {
            double s = 0.0;
            for (int d = 0; d < 9; ++d) {
                const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
                s += c[d] * f[(std::size_t)jy * nx + jx];
            }
            out[(std::size_t)gy * nx + gx] = s;
        }
    return out;
}

} // namespace ocb
