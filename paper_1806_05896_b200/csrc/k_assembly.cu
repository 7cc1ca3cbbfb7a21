// Device-side Q1 assembly into the 9-diagonal layout.
//
// The same element formulas as assembly.cpp (the reference's fem.cpp:35-106:
// 2x2 Gauss mass, stiffness and SUPG convection-diffusion elements, default
// wind fem.cpp:164-169, Dirichlet elimination fem.cpp:109-140), evaluated per
// NODE instead of per element: node i gathers the rows of its four elements in
// the host scatter's element order (ey, then ex, ascending), so every entry is
// accumulated from 0.0 in the same sequence as the host assembly. This file is
// compiled with -fmad=false, so products and sums round exactly as on the host
// (the only libm call, hypot in the SUPG parameter, may differ by an ulp).
#include "kernels.hpp"

namespace ocb {

namespace {

constexpr double kG = 0.57735026918962576;

struct Q1 {
    double a[4][4];
};

__device__ __forceinline__ void qpt(int q, double& xi, double& eta)
{
    // corner order SW, SE, NE, NW (fem.cpp:16-19)
    xi = (q == 0 || q == 3) ? -kG : kG;
    eta = (q < 2) ? -kG : kG;
}

__device__ __forceinline__ void shape(double xi, double eta, double N[4])
{
    N[0] = 0.25 * (1 - xi) * (1 - eta);
    N[1] = 0.25 * (1 + xi) * (1 - eta);
    N[2] = 0.25 * (1 + xi) * (1 + eta);
    N[3] = 0.25 * (1 - xi) * (1 + eta);
}

__device__ __forceinline__ void shape_grad(double xi, double eta, double G[4][2])
{
    G[0][0] = -0.25 * (1 - eta); G[0][1] = -0.25 * (1 - xi);
    G[1][0] = 0.25 * (1 - eta);  G[1][1] = -0.25 * (1 + xi);
    G[2][0] = 0.25 * (1 + eta);  G[2][1] = 0.25 * (1 + xi);
    G[3][0] = -0.25 * (1 + eta); G[3][1] = 0.25 * (1 - xi);
}

__device__ void element_mass(double h, Q1& m)
{
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) m.a[i][j] = 0.0;
    const double detj = h * h / 4.0;
    for (int q = 0; q < 4; ++q) {
        double xi, eta, N[4];
        qpt(q, xi, eta);
        shape(xi, eta, N);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) m.a[i][j] += N[i] * N[j] * detj;
    }
}

__device__ void element_stiffness(double h, Q1& k)
{
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) k.a[i][j] = 0.0;
    const double detj = h * h / 4.0;
    const double s = 2.0 / h;
    for (int q = 0; q < 4; ++q) {
        double xi, eta, G[4][2];
        qpt(q, xi, eta);
        shape_grad(xi, eta, G);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                k.a[i][j] += s * s * (G[i][0] * G[j][0] + G[i][1] * G[j][1]) * detj;
    }
}

__device__ __forceinline__ void wind(double x1, double x2, double w[2])
{
    w[0] = 2.0 * x2 * (1.0 - x1 * x1);
    w[1] = -2.0 * x1 * (1.0 - x2 * x2);
}

__device__ void element_convdiff(double h, int ex, int ey, double eps, Q1& a)
{
    const double x0 = ex * h, y0 = ey * h;
    const double detj = h * h / 4.0;
    const double s = 2.0 / h;
    element_stiffness(h, a);
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) a.a[i][j] *= eps;
    double wc[2];
    wind(x0 + 0.5 * h, y0 + 0.5 * h, wc);
    const double wnorm = hypot(wc[0], wc[1]);
    double delta = 0.0;
    if (wnorm > 1e-14) {
        const double peclet = wnorm * h / (2.0 * eps);
        delta = h / (2.0 * wnorm) * fmax(0.0, 1.0 - 1.0 / peclet);
    }
    for (int q = 0; q < 4; ++q) {
        double xi, eta, N[4], G[4][2], w[2];
        qpt(q, xi, eta);
        shape(xi, eta, N);
        shape_grad(xi, eta, G);
        const double xq = x0 + 0.5 * h * (xi + 1.0);
        const double yq = y0 + 0.5 * h * (eta + 1.0);
        wind(xq, yq, w);
        double wg[4];
        for (int i = 0; i < 4; ++i) wg[i] = s * (w[0] * G[i][0] + w[1] * G[i][1]);
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                a.a[i][j] += wg[j] * N[i] * detj;
                if (delta > 0.0) a.a[i][j] += delta * wg[j] * wg[i] * detj;
            }
    }
}

// what: 0 mass, 1 Poisson, 2 SUPG convection-diffusion, 3 partial-observation mass
__global__ void k_assemble9(int what, int level, double eps, double o0, double o1, double o2,
                            double o3, double* __restrict__ coef)
{
    const int nx = (1 << level) - 1;
    const long long n = (long long)nx * nx;
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const int gyi = (int)row / nx + 1, gxi = (int)row - (gyi - 1) * nx + 1; // 1-based
    const double h = 1.0 / double(1 << level);
    const int lx[4] = {0, 1, 1, 0}, ly[4] = {0, 0, 1, 1};
    double c[9];
    for (int d = 0; d < 9; ++d) c[d] = 0.0;
    Q1 a;
    if (what == 0 || what == 3) element_mass(h, a);
    else if (what == 1) element_stiffness(h, a);
    // the node's four elements in the host scatter order (ey, then ex, ascending)
    for (int e = 0; e < 4; ++e) {
        const int ex = gxi - 1 + (e & 1), ey = gyi - 1 + (e >> 1);
        if (what == 2) element_convdiff(h, ex, ey, eps, a);
        if (what == 3) {
            const double tol = 1e-12; // ObservationRegion::contains_box (grid.hpp:53-57)
            const double x0 = ex * h, x1 = (ex + 1) * h, y0 = ey * h, y1 = (ey + 1) * h;
            const bool in = x0 >= o0 - tol && x1 <= o1 + tol && y0 >= o2 - tol && y1 <= o3 + tol;
            if (!in) continue; // a zero element adds exact zeros
        }
        int i = 0; // local index of this node in element (ex, ey)
        for (int k = 0; k < 4; ++k)
            if (ex + lx[k] == gxi && ey + ly[k] == gyi) i = k;
        for (int j = 0; j < 4; ++j) {
            const int gxj = ex + lx[j], gyj = ey + ly[j];
            if (gxj < 1 || gxj > nx || gyj < 1 || gyj > nx) continue;
            const int d = (gyj - gyi + 1) * 3 + (gxj - gxi + 1);
            c[d] += a.a[i][j];
        }
    }
    for (int d = 0; d < 9; ++d) coef[d * n + row] = c[d];
}

// T(i, i + off(e)) = A(i + off(e), i), i.e. entry 8 - e of row j (transpose9)
__global__ void k_transpose9(int nx, const double* __restrict__ in, double* __restrict__ out)
{
    const long long n = (long long)nx * nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int gy = (int)i / nx, gx = (int)i - gy * nx;
    for (int e = 0; e < 9; ++e) {
        const int jx = gx + e % 3 - 1, jy = gy + e / 3 - 1;
        double v = 0.0;
        if (jx >= 0 && jx < nx && jy >= 0 && jy < nx) v = in[(8 - e) * n + (long long)jy * nx + jx];
        out[e * n + i] = v;
    }
}

// out = 1.0 * a + 1.0 * b entrywise (sparse_add over the 9-diagonal layout)
__global__ void k_add9(long long m, const double* __restrict__ a, const double* __restrict__ b,
                       double* __restrict__ out)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = 1.0 * a[i] + 1.0 * b[i];
}

} // namespace

void launch_assemble9(cudaStream_t s, int what, int level, double eps, const double* obs,
                      double* coef)
{
    const long long nx = (1 << level) - 1, n = nx * nx;
    note_launch();
    k_assemble9<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
        what, level, eps, obs ? obs[0] : 0.0, obs ? obs[1] : 0.0, obs ? obs[2] : 0.0,
        obs ? obs[3] : 0.0, coef);
}

void launch_transpose9(cudaStream_t s, int nx, const double* in, double* out)
{
    const long long n = (long long)nx * nx;
    note_launch();
    k_transpose9<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nx, in, out);
}

void launch_add9(cudaStream_t s, long long m, const double* a, const double* b, double* out)
{
    note_launch();
    k_add9<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, a, b, out);
}

} // namespace ocb
