// Eigen-free DenseFactor for the oracle build (TEST INFRASTRUCTURE ONLY).
//
// The reference implements optcon::DenseFactor (include/optcon/dense_eig.hpp:29-44)
// with Eigen::PartialPivLU (src/dense_eig.cpp:87-121). Eigen3 is not in this
// image, so the oracle links this restatement instead: a right-looking LU with
// partial (row) pivoting on the column of largest magnitude, which is the
// algorithm PartialPivLU documents. Results differ from Eigen's blocked kernel
// only by rounding. It is used by the reference for the level-2 (9x9) multigrid
// coarse solve (multigrid.cpp:107,113-116) and the dense verification solver.
#include "optcon/dense_eig.hpp"

#include <cmath>
#include <stdexcept>
#include <utility>
#include <vector>

namespace optcon {

struct DenseFactor::Impl {
    std::int32_t n = 0;
    std::vector<double> lu;          // column-major packed L\U
    std::vector<std::int32_t> perm;  // row permutation: row i of PA is row perm[i] of A

    void factor()
    {
        perm.resize(static_cast<std::size_t>(n));
        for (std::int32_t i = 0; i < n; ++i) perm[i] = i;
        auto at = [this](std::int32_t i, std::int32_t j) -> double& {
            return lu[static_cast<std::size_t>(j) * n + i];
        };
        for (std::int32_t k = 0; k < n; ++k) {
            std::int32_t piv = k;
            double best = std::abs(at(k, k));
            for (std::int32_t i = k + 1; i < n; ++i)
                if (std::abs(at(i, k)) > best) {
                    best = std::abs(at(i, k));
                    piv = i;
                }
            if (piv != k) {
                for (std::int32_t j = 0; j < n; ++j) std::swap(at(k, j), at(piv, j));
                std::swap(perm[k], perm[piv]);
            }
            const double p = at(k, k);
            if (p == 0.0) continue; // singular column: Eigen also proceeds
            for (std::int32_t i = k + 1; i < n; ++i) at(i, k) /= p;
            for (std::int32_t j = k + 1; j < n; ++j) {
                const double ukj = at(k, j);
                if (ukj == 0.0) continue;
                for (std::int32_t i = k + 1; i < n; ++i) at(i, j) -= at(i, k) * ukj;
            }
        }
    }
};

DenseFactor::DenseFactor(const SparseMatrix& A)
{
    if (A.rows() != A.cols()) throw std::invalid_argument("DenseFactor: matrix not square");
    if (A.rows() > kDenseVerificationCap)
        throw std::invalid_argument("DenseFactor: matrix exceeds the verification cap");
    impl_ = std::make_unique<Impl>();
    const std::int32_t n = A.rows();
    impl_->n = n;
    impl_->lu.assign(static_cast<std::size_t>(n) * n, 0.0);
    for (std::int32_t i = 0; i < n; ++i)
        for (std::int32_t k = A.row_ptr()[i]; k < A.row_ptr()[i + 1]; ++k)
            impl_->lu[static_cast<std::size_t>(A.col_idx()[k]) * n + i] = A.values()[k];
    impl_->factor();
}

DenseFactor::DenseFactor(std::vector<double> data, std::int32_t n)
{
    if (static_cast<std::size_t>(n) * static_cast<std::size_t>(n) != data.size())
        throw std::invalid_argument("DenseFactor: bad data size");
    impl_ = std::make_unique<Impl>();
    impl_->n = n;
    impl_->lu = std::move(data);
    impl_->factor();
}

DenseFactor::~DenseFactor() = default;
DenseFactor::DenseFactor(DenseFactor&&) noexcept = default;
DenseFactor& DenseFactor::operator=(DenseFactor&&) noexcept = default;

Vector DenseFactor::solve(const Vector& rhs) const
{
    const std::int32_t n = impl_->n;
    if (static_cast<std::int32_t>(rhs.size()) != n)
        throw std::invalid_argument("DenseFactor::solve: dimension mismatch");
    const auto& lu = impl_->lu;
    Vector x(static_cast<std::size_t>(n));
    for (std::int32_t i = 0; i < n; ++i) x[i] = rhs[impl_->perm[i]];
    for (std::int32_t i = 0; i < n; ++i)
        for (std::int32_t k = 0; k < i; ++k) x[i] -= lu[static_cast<std::size_t>(k) * n + i] * x[k];
    for (std::int32_t i = n - 1; i >= 0; --i) {
        for (std::int32_t k = i + 1; k < n; ++k) x[i] -= lu[static_cast<std::size_t>(k) * n + i] * x[k];
        x[i] /= lu[static_cast<std::size_t>(i) * n + i];
    }
    return x;
}

std::int32_t DenseFactor::size() const { return impl_->n; }

} // namespace optcon
