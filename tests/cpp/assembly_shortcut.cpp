// The constant-stencil shortcuts used by the problem setup are bitwise the
// full host assembly (assembly.hpp: stencil9, lumped_from_stencil,
// apply_stencil vs assemble_mass9 / assemble_poisson9 / lumped_diag).
#include "../../paper_1806_05896_b200/csrc/assembly.hpp"

#include <cstdio>
#include <cstring>

int main()
{
    using namespace ocb;
    int bad = 0;
    for (int level = 2; level <= 10; ++level) {
        const int nx = level_nx(level);
        const long long n = (long long)nx * nx, mid = (long long)(nx / 2) * nx + nx / 2;
        const std::vector<double> M = assemble_mass9(level), L = assemble_poisson9(level);
        double cM[9], cL[9];
        stencil9(0, level, cM);
        stencil9(1, level, cL);
        for (int d = 0; d < 9; ++d) {
            if (memcmp(&cM[d], &M[d * n + mid], 8) || memcmp(&cL[d], &L[d * n + mid], 8)) {
                std::printf("level %d entry %d differs\n", level, d);
                ++bad;
            }
        }
        const std::vector<double> a = lumped_diag(level), b = lumped_from_stencil(cM, level);
        if (memcmp(a.data(), b.data(), a.size() * 8)) {
            std::printf("level %d lumped differs\n", level);
            ++bad;
        }
        std::vector<double> f(n);
        for (long long i = 0; i < n; ++i) f[i] = 0.25 + 1e-3 * (double)(i % 97);
        const std::vector<double> mf = apply_stencil(cM, level, f);
        for (long long i = 0; i < n; ++i) {
            const int gx = (int)(i % nx), gy = (int)(i / nx);
            double s = 0.0;
            for (int d = 0; d < 9; ++d) {
                const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
                s += M[d * n + i] * f[(long long)jy * nx + jx];
            }
            if (memcmp(&s, &mf[i], 8)) {
                std::printf("level %d M f differs at %lld\n", level, i);
                ++bad;
                break;
            }
        }
    }
    std::printf(bad ? "FAIL\n" : "ok\n");
    return bad ? 1 : 0;
}
