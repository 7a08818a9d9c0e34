#pragma once
// Eigen-free dense types of the drop-in API (reference: types.hpp:1-20, which
// aliases Eigen).  Eigen is not a dependency of the B200 build; these types keep
// the subset of the Eigen interface the reference callers use: (i,j) access,
// rows()/cols()/size(), data(), resize(), row-major storage, Vec3 arithmetic
// with x()/y()/z(), norm(), squaredNorm(), dot(), cross().

#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <vector>

namespace pswarm {

using Index = std::int64_t;

/// Components per Cartesian state (types.hpp:18).
inline constexpr Index state_dim = 6;

/// Dense row-major matrix (types.hpp:11): one time node per contiguous row.
class Mat {
public:
    Mat() = default;
    Mat(Index rows, Index cols) : rows_(rows), cols_(cols), v_(static_cast<std::size_t>(rows * cols), 0.0) {}
    static Mat Zero(Index rows, Index cols) { return Mat(rows, cols); }
    static Mat Constant(Index rows, Index cols, double x) {
        Mat m(rows, cols);
        for (auto& e : m.v_) e = x;
        return m;
    }
    double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i * cols_ + j)]; }
    double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(i * cols_ + j)]; }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double* row_data(Index i) { return v_.data() + i * cols_; }
    const double* row_data(Index i) const { return v_.data() + i * cols_; }
    void resize(Index rows, Index cols) {
        rows_ = rows;
        cols_ = cols;
        v_.assign(static_cast<std::size_t>(rows * cols), 0.0);
    }
    bool allFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    bool operator==(const Mat& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && v_ == o.v_; }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<double> v_;
};

/// Dense column vector (Eigen::VectorXd subset).
class Vec {
public:
    Vec() = default;
    explicit Vec(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
    Vec(std::initializer_list<double> xs) : v_(xs) {}
    double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    Index size() const { return static_cast<Index>(v_.size()); }
    void resize(Index n) { v_.assign(static_cast<std::size_t>(n), 0.0); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    bool operator==(const Vec& o) const { return v_ == o.v_; }

private:
    std::vector<double> v_;
};

/// Row vector (Eigen::Matrix<double, 1, Dynamic> subset); same storage as Vec.
using RowVec = Vec;

/// 3-vector (Eigen::Vector3d subset).
class Vec3 {
public:
    constexpr Vec3() = default;
    constexpr Vec3(double x, double y, double z) : e_{x, y, z} {}
    static constexpr Vec3 Zero() { return {}; }
    double& x() { return e_[0]; }
    double& y() { return e_[1]; }
    double& z() { return e_[2]; }
    double x() const { return e_[0]; }
    double y() const { return e_[1]; }
    double z() const { return e_[2]; }
    double& operator[](Index i) { return e_[i]; }
    double operator[](Index i) const { return e_[i]; }
    double& operator()(Index i) { return e_[i]; }
    double operator()(Index i) const { return e_[i]; }
    double squaredNorm() const { return e_[0] * e_[0] + e_[1] * e_[1] + e_[2] * e_[2]; }
    double norm() const { return std::sqrt(squaredNorm()); }
    double dot(const Vec3& o) const { return e_[0] * o.e_[0] + e_[1] * o.e_[1] + e_[2] * o.e_[2]; }
    Vec3 cross(const Vec3& o) const {
        return {e_[1] * o.e_[2] - e_[2] * o.e_[1], e_[2] * o.e_[0] - e_[0] * o.e_[2], e_[0] * o.e_[1] - e_[1] * o.e_[0]};
    }
    bool allFinite() const { return std::isfinite(e_[0]) && std::isfinite(e_[1]) && std::isfinite(e_[2]); }
    Vec3& operator+=(const Vec3& o) {
        for (int i = 0; i < 3; ++i) e_[i] += o.e_[i];
        return *this;
    }
    Vec3& operator-=(const Vec3& o) {
        for (int i = 0; i < 3; ++i) e_[i] -= o.e_[i];
        return *this;
    }
    bool operator==(const Vec3& o) const { return e_[0] == o.e_[0] && e_[1] == o.e_[1] && e_[2] == o.e_[2]; }

private:
    double e_[3] = {0.0, 0.0, 0.0};
};

inline Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
inline Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
inline Vec3 operator-(const Vec3& a) { return {-a.x(), -a.y(), -a.z()}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a.x(), s * a.y(), s * a.z()}; }
inline Vec3 operator*(const Vec3& a, double s) { return s * a; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x() / s, a.y() / s, a.z() / s}; }

}  // namespace pswarm
