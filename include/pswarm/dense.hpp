#pragma once
// Dense linear-algebra subset used by the reference's batch-propagation API.
//
// The reference aliases Eigen (proj/include/pswarm/types.hpp:3-15): Mat is a
// row-major dynamic Matrix, Vec/RowVec dynamic vectors, Vec3 a Vector3d, and
// oracle.hpp:18 adds State6 = Matrix<double, 6, 1>.  Eigen is not a dependency
// of the B200 build, so this header provides the part of Eigen's interface that
// reference code calls (proj/include/pswarm/*.hpp and proj/tests/*.cpp), with the
// same semantics:
//
//  * Matrix<Scalar, Rows, Cols, Options> with Dynamic sizes, fixed-size storage on
//    the stack, row- or column-major storage, Zero/Ones/Constant/Identity/UnitX..;
//  * writable strided views: row, col, block, head/tail/segment (static and
//    dynamic), top/middle/bottomRows, left/middle/rightCols, transpose, Map;
//  * element-wise + - and scalar * /, the matrix product (a register-blocked
//    SSE2 kernel on row-major operands), comma initialisation (m << a, b, ...),
//    rowwise() broadcasts, noalias(), array() comparisons and element-wise ops,
//    reductions (sum, maxCoeff, norm, squaredNorm, dot, cross, allFinite, ...);
//  * assignment between row and column vectors of equal size (Eigen's implicit
//    vector transposition), reference semantics for views (assigning to a view
//    writes through; copying a view object rebinds nothing).
//
// Arithmetic is evaluated eagerly into plain matrices; views are the only lazy
// objects (they never own memory, like Eigen's Block/Map/Transpose).  include/
// pswarm/types.hpp aliases these types, unless PSWARM_USE_EIGEN selects Eigen
// itself.  oracle/eigen_shim/Eigen/Dense maps namespace Eigen onto this header to
// compile the reference's own headers unchanged (test infrastructure).
#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace pswarm::dense {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
inline constexpr int Infinity = -1;
enum StorageOptions : int { ColMajor = 0, RowMajor = 0x1, AutoAlign = 0, DontAlign = 0x2 };

#define PSWARM_DENSE_CHECK(cond, msg) \
    do {                              \
        if (!(cond)) throw std::logic_error(std::string("pswarm::dense: ") + (msg)); \
    } while (0)

template <class S, int R, int C, int Opt = ((R == 1 && C != 1) ? RowMajor : ColMajor), int MR = R, int MC = C>
class Matrix;
template <class S, int R, int C, bool Const>
class View;
template <class Derived>
class ArrayView;

template <class T>
struct traits;

namespace detail {
constexpr int prod_size(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : a * b; }
constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }
constexpr int plain_opt(int r, int c) { return (r == 1 && c != 1) ? RowMajor : (c == 1 && r != 1) ? ColMajor : RowMajor; }
}  // namespace detail

/// Plain (owning) type of an expression with compile-time shape R x C.
template <class S, int R, int C>
using Plain = Matrix<S, R, C, detail::plain_opt(R, C)>;

template <class Derived>
class RowwiseProxy;

// ---------------------------------------------------------------------------
// DenseBase: read-only interface of every dense object (all are strided
// direct-access: data() + rows/cols + row/col strides).
template <class Derived>
class DenseBase {
public:
    using Scalar = typename traits<Derived>::Scalar;
    static constexpr int RowsAtCompileTime = traits<Derived>::Rows;
    static constexpr int ColsAtCompileTime = traits<Derived>::Cols;
    static constexpr int SizeAtCompileTime = detail::prod_size(RowsAtCompileTime, ColsAtCompileTime);
    static constexpr bool IsVectorAtCompileTime = RowsAtCompileTime == 1 || ColsAtCompileTime == 1;
    using PlainObject = Plain<Scalar, RowsAtCompileTime, ColsAtCompileTime>;
    using ConstView = View<Scalar, RowsAtCompileTime, ColsAtCompileTime, true>;

    const Derived& derived() const { return *static_cast<const Derived*>(this); }
    Derived& derived() { return *static_cast<Derived*>(this); }

    Index rows() const { return derived().rows_(); }
    Index cols() const { return derived().cols_(); }
    Index size() const { return rows() * cols(); }
    Index rstride() const { return derived().rstride_(); }
    Index cstride() const { return derived().cstride_(); }
    const Scalar* data() const { return derived().cdata_(); }
    bool is_vector() const { return rows() == 1 || cols() == 1; }

    Scalar coeff(Index i, Index j) const { return data()[i * rstride() + j * cstride()]; }
    /// linear coefficient of a vector (either orientation)
    Scalar coeff(Index k) const { return rows() == 1 ? coeff(0, k) : coeff(k, 0); }
    Scalar operator()(Index i, Index j) const { return coeff(i, j); }
    Scalar operator()(Index k) const { return coeff(k); }
    Scalar operator[](Index k) const { return coeff(k); }
    Scalar x() const { return coeff(0); }
    Scalar y() const { return coeff(1); }
    Scalar z() const { return coeff(2); }
    Scalar w() const { return coeff(3); }

    // ---- views (read-only)
    View<Scalar, 1, ColsAtCompileTime, true> row(Index i) const {
        return {data() + i * rstride(), 1, cols(), rstride(), cstride()};
    }
    View<Scalar, RowsAtCompileTime, 1, true> col(Index j) const {
        return {data() + j * cstride(), rows(), 1, rstride(), cstride()};
    }
    View<Scalar, Dynamic, Dynamic, true> block(Index i, Index j, Index r, Index c) const {
        return {data() + i * rstride() + j * cstride(), r, c, rstride(), cstride()};
    }
    template <int BR, int BC>
    View<Scalar, BR, BC, true> block(Index i, Index j) const {
        return {data() + i * rstride() + j * cstride(), BR, BC, rstride(), cstride()};
    }
    View<Scalar, Dynamic, ColsAtCompileTime, true> topRows(Index n) const { return middleRows(0, n); }
    View<Scalar, Dynamic, ColsAtCompileTime, true> bottomRows(Index n) const { return middleRows(rows() - n, n); }
    View<Scalar, Dynamic, ColsAtCompileTime, true> middleRows(Index i, Index n) const {
        return {data() + i * rstride(), n, cols(), rstride(), cstride()};
    }
    View<Scalar, RowsAtCompileTime, Dynamic, true> leftCols(Index n) const { return middleCols(0, n); }
    View<Scalar, RowsAtCompileTime, Dynamic, true> rightCols(Index n) const { return middleCols(cols() - n, n); }
    View<Scalar, RowsAtCompileTime, Dynamic, true> middleCols(Index j, Index n) const {
        return {data() + j * cstride(), rows(), n, rstride(), cstride()};
    }
    View<Scalar, ColsAtCompileTime, RowsAtCompileTime, true> transpose() const {
        return {data(), cols(), rows(), cstride(), rstride()};
    }
    auto segment(Index i, Index n) const { return vseg<Dynamic>(i, n); }
    auto head(Index n) const { return vseg<Dynamic>(0, n); }
    auto tail(Index n) const { return vseg<Dynamic>(size() - n, n); }
    template <int N>
    auto segment(Index i) const { return vseg<N>(i, N); }
    template <int N>
    auto head() const { return vseg<N>(0, N); }
    template <int N>
    auto tail() const { return vseg<N>(size() - N, N); }

    // ---- evaluation
    PlainObject eval() const { return PlainObject(derived()); }
    ArrayView<Derived> array() const { return ArrayView<Derived>(derived()); }
    const Derived& matrix() const { return derived(); }

    // ---- reductions
    template <class F>
    void visit(F&& f) const {
        const Index r = rows(), c = cols(), rs = rstride(), cs = cstride();
        const Scalar* p = data();
        if (cs == 1) {
            for (Index i = 0; i < r; ++i)
                for (Index j = 0; j < c; ++j) f(p[i * rs + j]);
        } else {
            for (Index j = 0; j < c; ++j)
                for (Index i = 0; i < r; ++i) f(p[i * rs + j * cs]);
        }
    }
    Scalar sum() const {
        Scalar s = 0;
        visit([&](Scalar v) { s += v; });
        return s;
    }
    Scalar prod() const {
        Scalar s = 1;
        visit([&](Scalar v) { s *= v; });
        return s;
    }
    Scalar mean() const { return sum() / static_cast<Scalar>(size()); }
    Scalar squaredNorm() const {
        Scalar s = 0;
        visit([&](Scalar v) { s += v * v; });
        return s;
    }
    Scalar norm() const { return std::sqrt(squaredNorm()); }
    Scalar stableNorm() const { return norm(); }
    template <int P>
    Scalar lpNorm() const {
        if constexpr (P == Infinity) {
            Scalar m = 0;
            visit([&](Scalar v) { m = std::max(m, std::abs(v)); });
            return m;
        } else if constexpr (P == 1) {
            Scalar s = 0;
            visit([&](Scalar v) { s += std::abs(v); });
            return s;
        } else {
            static_assert(P == 2, "lpNorm<1|2|Infinity> only");
            return norm();
        }
    }
    Scalar maxCoeff() const {
        PSWARM_DENSE_CHECK(size() > 0, "maxCoeff of an empty object");
        Scalar m = coeff(0, 0);
        visit([&](Scalar v) { m = (v > m) ? v : m; });
        return m;
    }
    Scalar minCoeff() const {
        PSWARM_DENSE_CHECK(size() > 0, "minCoeff of an empty object");
        Scalar m = coeff(0, 0);
        visit([&](Scalar v) { m = (v < m) ? v : m; });
        return m;
    }
    template <class I>
    Scalar maxCoeff(I* index) const {
        PSWARM_DENSE_CHECK(size() > 0 && is_vector(), "maxCoeff(index) needs a non-empty vector");
        Index best = 0;
        for (Index k = 1; k < size(); ++k)
            if (coeff(k) > coeff(best)) best = k;
        *index = static_cast<I>(best);
        return coeff(best);
    }
    template <class I>
    Scalar minCoeff(I* index) const {
        PSWARM_DENSE_CHECK(size() > 0 && is_vector(), "minCoeff(index) needs a non-empty vector");
        Index best = 0;
        for (Index k = 1; k < size(); ++k)
            if (coeff(k) < coeff(best)) best = k;
        *index = static_cast<I>(best);
        return coeff(best);
    }
    bool allFinite() const {
        bool ok = true;
        visit([&](Scalar v) { ok = ok && std::isfinite(v); });
        return ok;
    }
    bool hasNaN() const {
        bool nan = false;
        visit([&](Scalar v) { nan = nan || std::isnan(v); });
        return nan;
    }
    bool isZero(Scalar prec = Scalar(1e-12)) const { return lpNorm<Infinity>() <= prec; }
    template <class O>
    Scalar dot(const DenseBase<O>& o) const {
        PSWARM_DENSE_CHECK(size() == o.size() && is_vector() && o.is_vector(), "dot: size mismatch");
        Scalar s = 0;
        for (Index k = 0; k < size(); ++k) s += coeff(k) * o.coeff(k);
        return s;
    }
    template <class O>
    PlainObject cross(const DenseBase<O>& o) const {
        PSWARM_DENSE_CHECK(size() == 3 && o.size() == 3, "cross: 3-vectors only");
        PlainObject out(derived());
        out.coeffRef(0) = coeff(1) * o.coeff(2) - coeff(2) * o.coeff(1);
        out.coeffRef(1) = coeff(2) * o.coeff(0) - coeff(0) * o.coeff(2);
        out.coeffRef(2) = coeff(0) * o.coeff(1) - coeff(1) * o.coeff(0);
        return out;
    }
    PlainObject normalized() const {
        PlainObject out(derived());
        const Scalar n = norm();
        if (n > 0) out /= n;
        return out;
    }
    template <class F>
    PlainObject unaryExpr(F&& f) const {
        PlainObject out(derived());
        out.apply([&](Scalar& v) { v = f(v); });
        return out;
    }
    PlainObject cwiseAbs() const {
        return unaryExpr([](Scalar v) { return std::abs(v); });
    }
    PlainObject cwiseAbs2() const {
        return unaryExpr([](Scalar v) { return v * v; });
    }
    PlainObject cwiseSqrt() const {
        return unaryExpr([](Scalar v) { return std::sqrt(v); });
    }
    template <class O, class F>
    PlainObject binaryExpr(const DenseBase<O>& o, F&& f) const;
    template <class O>
    PlainObject cwiseMax(const DenseBase<O>& o) const {
        return binaryExpr(o, [](Scalar a, Scalar b) { return std::max(a, b); });
    }
    template <class O>
    PlainObject cwiseMin(const DenseBase<O>& o) const {
        return binaryExpr(o, [](Scalar a, Scalar b) { return std::min(a, b); });
    }
    template <class O>
    PlainObject cwiseProduct(const DenseBase<O>& o) const {
        return binaryExpr(o, [](Scalar a, Scalar b) { return a * b; });
    }
    template <class O>
    PlainObject cwiseQuotient(const DenseBase<O>& o) const {
        return binaryExpr(o, [](Scalar a, Scalar b) { return a / b; });
    }
    PlainObject cwiseMax(Scalar s) const {
        return unaryExpr([s](Scalar v) { return std::max(v, s); });
    }
    PlainObject cwiseMin(Scalar s) const {
        return unaryExpr([s](Scalar v) { return std::min(v, s); });
    }
    template <class O>
    bool isApprox(const DenseBase<O>& o, Scalar prec = Scalar(1e-12)) const {
        Scalar d = 0, a = 0, b = 0;
        PSWARM_DENSE_CHECK(rows() == o.rows() && cols() == o.cols(), "isApprox: shape mismatch");
        for (Index i = 0; i < rows(); ++i)
            for (Index j = 0; j < cols(); ++j) {
                const Scalar x = coeff(i, j), y = o.coeff(i, j);
                d += (x - y) * (x - y);
                a += x * x;
                b += y * y;
            }
        return std::sqrt(d) <= prec * std::sqrt(std::min(a, b));
    }

private:
    template <int N>
    auto vseg(Index i, Index n) const {
        PSWARM_DENSE_CHECK(is_vector(), "segment/head/tail on a non-vector");
        constexpr bool row_vec = RowsAtCompileTime == 1;
        if constexpr (row_vec) {
            return View<Scalar, 1, N, true>{data() + i * cstride(), 1, n, rstride(), cstride()};
        } else {
            if (rows() == 1)  // dynamic-shaped object that is a row at run time
                return View<Scalar, N, 1, true>{data() + i * cstride(), n, 1, cstride(), rstride()};
            return View<Scalar, N, 1, true>{data() + i * rstride(), n, 1, rstride(), cstride()};
        }
    }
};

// ---------------------------------------------------------------------------
// DenseWritable: mutating interface (plain matrices and non-const views).
template <class Derived>
class DenseWritable : public DenseBase<Derived> {
public:
    using Base = DenseBase<Derived>;
    using typename Base::Scalar;
    using Base::cols;
    using Base::cstride;
    using Base::data;
    using Base::derived;
    using Base::rows;
    using Base::rstride;
    using Base::size;
    static constexpr int RowsAtCompileTime = Base::RowsAtCompileTime;
    static constexpr int ColsAtCompileTime = Base::ColsAtCompileTime;

    Scalar* data() { return derived().mdata_(); }
    Scalar& coeffRef(Index i, Index j) { return data()[i * rstride() + j * cstride()]; }
    Scalar& coeffRef(Index k) { return rows() == 1 ? coeffRef(0, k) : coeffRef(k, 0); }
    using Base::operator();
    using Base::operator[];
    Scalar& operator()(Index i, Index j) { return coeffRef(i, j); }
    Scalar& operator()(Index k) { return coeffRef(k); }
    Scalar& operator[](Index k) { return coeffRef(k); }
    using Base::x;
    using Base::y;
    using Base::z;
    using Base::w;
    Scalar& x() { return coeffRef(0); }
    Scalar& y() { return coeffRef(1); }
    Scalar& z() { return coeffRef(2); }
    Scalar& w() { return coeffRef(3); }

    template <class F>
    void apply(F&& f) {
        const Index r = rows(), c = cols(), rs = rstride(), cs = cstride();
        Scalar* p = data();
        if (cs == 1) {
            for (Index i = 0; i < r; ++i)
                for (Index j = 0; j < c; ++j) f(p[i * rs + j]);
        } else {
            for (Index j = 0; j < c; ++j)
                for (Index i = 0; i < r; ++i) f(p[i * rs + j * cs]);
        }
    }

    // ---- writable views
    using Base::block;
    using Base::col;
    using Base::head;
    using Base::leftCols;
    using Base::middleCols;
    using Base::middleRows;
    using Base::rightCols;
    using Base::row;
    using Base::segment;
    using Base::tail;
    using Base::topRows;
    using Base::bottomRows;
    using Base::transpose;
    View<Scalar, 1, ColsAtCompileTime, false> row(Index i) {
        return {data() + i * rstride(), 1, cols(), rstride(), cstride()};
    }
    View<Scalar, RowsAtCompileTime, 1, false> col(Index j) {
        return {data() + j * cstride(), rows(), 1, rstride(), cstride()};
    }
    View<Scalar, Dynamic, Dynamic, false> block(Index i, Index j, Index r, Index c) {
        return {data() + i * rstride() + j * cstride(), r, c, rstride(), cstride()};
    }
    template <int BR, int BC>
    View<Scalar, BR, BC, false> block(Index i, Index j) {
        return {data() + i * rstride() + j * cstride(), BR, BC, rstride(), cstride()};
    }
    View<Scalar, Dynamic, ColsAtCompileTime, false> topRows(Index n) { return middleRows(0, n); }
    View<Scalar, Dynamic, ColsAtCompileTime, false> bottomRows(Index n) { return middleRows(rows() - n, n); }
    View<Scalar, Dynamic, ColsAtCompileTime, false> middleRows(Index i, Index n) {
        return {data() + i * rstride(), n, cols(), rstride(), cstride()};
    }
    View<Scalar, RowsAtCompileTime, Dynamic, false> leftCols(Index n) { return middleCols(0, n); }
    View<Scalar, RowsAtCompileTime, Dynamic, false> rightCols(Index n) { return middleCols(cols() - n, n); }
    View<Scalar, RowsAtCompileTime, Dynamic, false> middleCols(Index j, Index n) {
        return {data() + j * cstride(), rows(), n, rstride(), cstride()};
    }
    View<Scalar, ColsAtCompileTime, RowsAtCompileTime, false> transpose() {
        return {data(), cols(), rows(), cstride(), rstride()};
    }
    auto segment(Index i, Index n) { return vseg<Dynamic>(i, n); }
    auto head(Index n) { return vseg<Dynamic>(0, n); }
    auto tail(Index n) { return vseg<Dynamic>(size() - n, n); }
    template <int N>
    auto segment(Index i) { return vseg<N>(i, N); }
    template <int N>
    auto head() { return vseg<N>(0, N); }
    template <int N>
    auto tail() { return vseg<N>(size() - N, N); }

    Derived& noalias() { return derived(); }
    RowwiseProxy<Derived> rowwise() { return RowwiseProxy<Derived>(derived()); }

    // ---- fills
    Derived& setConstant(Scalar v) {
        apply([v](Scalar& x) { x = v; });
        return derived();
    }
    Derived& fill(Scalar v) { return setConstant(v); }
    Derived& setZero() { return setConstant(Scalar(0)); }
    Derived& setOnes() { return setConstant(Scalar(1)); }
    Derived& setIdentity() {
        setZero();
        for (Index k = 0; k < std::min(rows(), cols()); ++k) coeffRef(k, k) = Scalar(1);
        return derived();
    }

    // ---- element-wise compound assignment
    template <class O>
    Derived& operator+=(const DenseBase<O>& o) {
        zip(o, [](Scalar& a, Scalar b) { a += b; });
        return derived();
    }
    template <class O>
    Derived& operator-=(const DenseBase<O>& o) {
        zip(o, [](Scalar& a, Scalar b) { a -= b; });
        return derived();
    }
    Derived& operator*=(Scalar s) {
        apply([s](Scalar& x) { x *= s; });
        return derived();
    }
    Derived& operator/=(Scalar s) {
        apply([s](Scalar& x) { x /= s; });
        return derived();
    }

    /// element copy from any dense object of the same shape (vectors: any orientation)
    template <class O>
    void assign_from(const DenseBase<O>& o) {
        zip(o, [](Scalar& a, Scalar b) { a = b; });
    }

    template <class O, class F>
    void zip(const DenseBase<O>& o, F&& f) {
        const Index r = rows(), c = cols();
        if (r == o.rows() && c == o.cols()) {
            const Index rs = rstride(), cs = cstride(), ors = o.rstride(), ocs = o.cstride();
            Scalar* p = data();
            const Scalar* q = o.data();
            if (cs == 1 && ocs == 1) {
                for (Index i = 0; i < r; ++i) {
                    Scalar* pr = p + i * rs;
                    const Scalar* qr = q + i * ors;
                    for (Index j = 0; j < c; ++j) f(pr[j], qr[j]);
                }
            } else {
                for (Index i = 0; i < r; ++i)
                    for (Index j = 0; j < c; ++j) f(p[i * rs + j * cs], q[i * ors + j * ocs]);
            }
        } else {
            PSWARM_DENSE_CHECK(this->is_vector() && o.is_vector() && size() == o.size(),
                               "shape mismatch (" + std::to_string(r) + "x" + std::to_string(c) + " vs " +
                                   std::to_string(o.rows()) + "x" + std::to_string(o.cols()) + ")");
            for (Index k = 0; k < size(); ++k) f(coeffRef(k), o.coeff(k));
        }
    }

private:
    template <int N>
    auto vseg(Index i, Index n) {
        PSWARM_DENSE_CHECK(this->is_vector(), "segment/head/tail on a non-vector");
        if constexpr (RowsAtCompileTime == 1) {
            return View<Scalar, 1, N, false>{data() + i * cstride(), 1, n, rstride(), cstride()};
        } else {
            if (rows() == 1)
                return View<Scalar, N, 1, false>{data() + i * cstride(), n, 1, cstride(), rstride()};
            return View<Scalar, N, 1, false>{data() + i * rstride(), n, 1, rstride(), cstride()};
        }
    }
};

// ---------------------------------------------------------------------------
// Comma initialiser: m << a, b, c  (scalars and dense blocks, row-major fill).
template <class Derived>
class CommaInitializer {
public:
    using Scalar = typename traits<Derived>::Scalar;
    explicit CommaInitializer(Derived& d) : d_(d) {}
    CommaInitializer(CommaInitializer&& o) noexcept : d_(o.d_), row_(o.row_), col_(o.col_), h_(o.h_) { o.done_ = true; }
    CommaInitializer& operator,(Scalar v) {
        put_scalar(v);
        return *this;
    }
    template <class O>
    CommaInitializer& operator,(const DenseBase<O>& o) {
        put_block(o);
        return *this;
    }
    void put_scalar(Scalar v) {
        advance_row();
        PSWARM_DENSE_CHECK(row_ < d_.rows() && col_ < d_.cols(), "too many coefficients passed to operator<<");
        d_.coeffRef(row_, col_) = v;
        ++col_;
        h_ = 1;
    }
    template <class O>
    void put_block(const DenseBase<O>& o) {
        if (o.size() == 0) return;
        advance_row();
        Index br = o.rows(), bc = o.cols();
        if (d_.cols() == 1 && br == 1 && bc > 1) {  // row block into a column vector: transposed fill
            PSWARM_DENSE_CHECK(row_ + bc <= d_.rows(), "too many coefficients passed to operator<<");
            for (Index k = 0; k < bc; ++k) d_.coeffRef(row_ + k, 0) = o.coeff(0, k);
            col_ = 1;
            h_ = bc;
            return;
        }
        if (d_.rows() == 1 && bc == 1 && br > 1) {  // column block into a row vector
            PSWARM_DENSE_CHECK(col_ + br <= d_.cols(), "too many coefficients passed to operator<<");
            for (Index k = 0; k < br; ++k) d_.coeffRef(0, col_ + k) = o.coeff(k, 0);
            col_ += br;
            h_ = 1;
            return;
        }
        PSWARM_DENSE_CHECK(row_ + br <= d_.rows() && col_ + bc <= d_.cols(), "too many coefficients passed to operator<<");
        for (Index i = 0; i < br; ++i)
            for (Index j = 0; j < bc; ++j) d_.coeffRef(row_ + i, col_ + j) = o.coeff(i, j);
        col_ += bc;
        h_ = br;
    }
    ~CommaInitializer() = default;
    Derived& finished() {
        done_ = true;
        return d_;
    }

private:
    void advance_row() {
        if (col_ == d_.cols() && d_.cols() > 0) {
            row_ += h_;
            col_ = 0;
            h_ = 1;
        }
    }
    Derived& d_;
    Index row_ = 0, col_ = 0, h_ = 1;
    bool done_ = false;
};

template <class D>
CommaInitializer<D> operator<<(DenseWritable<D>& d, typename traits<D>::Scalar v) {
    CommaInitializer<D> ci(d.derived());
    ci.put_scalar(v);
    return ci;
}
template <class D>
CommaInitializer<D> operator<<(DenseWritable<D>&& d, typename traits<D>::Scalar v) {
    return operator<<(static_cast<DenseWritable<D>&>(d), v);
}
template <class D, class O>
CommaInitializer<D> operator<<(DenseWritable<D>& d, const DenseBase<O>& o) {
    CommaInitializer<D> ci(d.derived());
    ci.put_block(o);
    return ci;
}
template <class D, class O>
CommaInitializer<D> operator<<(DenseWritable<D>&& d, const DenseBase<O>& o) {
    return operator<<(static_cast<DenseWritable<D>&>(d), o);
}

// ---------------------------------------------------------------------------
// View: strided, non-owning (Eigen's Block / Map / Transpose).
template <class S, int R, int C, bool Const>
struct traits<View<S, R, C, Const>> {
    using Scalar = S;
    static constexpr int Rows = R;
    static constexpr int Cols = C;
};

template <class S, int R, int C, bool Const>
class View : public std::conditional_t<Const, DenseBase<View<S, R, C, Const>>, DenseWritable<View<S, R, C, Const>>> {
public:
    using Ptr = std::conditional_t<Const, const S*, S*>;
    View(Ptr p, Index r, Index c, Index rs, Index cs) : p_(p), r_(r), c_(c), rs_(rs), cs_(cs) {}
    View(const View&) = default;
    /// a writable view converts to its read-only form
    template <bool C2 = Const, class = std::enable_if_t<C2>>
    View(const View<S, R, C, false>& o) : View(o.data(), o.rows(), o.cols(), o.rstride(), o.cstride()) {}

    // assignment writes through (Eigen semantics)
    View& operator=(const View& o) {
        static_assert(!Const, "assignment to a read-only view");
        this->assign_from(o);
        return *this;
    }
    template <class O>
    View& operator=(const DenseBase<O>& o) {
        static_assert(!Const, "assignment to a read-only view");
        this->assign_from(o);
        return *this;
    }

    Index rows_() const { return r_; }
    Index cols_() const { return c_; }
    Index rstride_() const { return rs_; }
    Index cstride_() const { return cs_; }
    const S* cdata_() const { return p_; }
    S* mdata_() { return const_cast<S*>(p_); }

private:
    Ptr p_;
    Index r_, c_, rs_, cs_;
};

// ---------------------------------------------------------------------------
// Matrix: owning storage.
template <class S, int R, int C, int Opt, int MR, int MC>
struct traits<Matrix<S, R, C, Opt, MR, MC>> {
    using Scalar = S;
    static constexpr int Rows = R;
    static constexpr int Cols = C;
};

namespace detail {
template <class S, int R, int C>
struct Storage {  // fixed size: on the stack, zero-initialised
    std::array<S, static_cast<std::size_t>(R * C)> a{};
    S* ptr() { return a.data(); }
    const S* ptr() const { return a.data(); }
    Index rows() const { return R; }
    Index cols() const { return C; }
    void resize(Index r, Index c) {
        PSWARM_DENSE_CHECK(r == R && c == C, "resize of a fixed-size matrix");
    }
};
template <class S>
struct DynStorage {
    std::unique_ptr<S[]> p;
    Index r = 0, c = 0, cap = 0;
    DynStorage() = default;
    DynStorage(const DynStorage& o) : r(o.r), c(o.c), cap(o.r * o.c) {
        if (cap) {
            p.reset(new S[static_cast<std::size_t>(cap)]);
            std::memcpy(p.get(), o.p.get(), sizeof(S) * static_cast<std::size_t>(cap));
        }
    }
    DynStorage(DynStorage&& o) noexcept : p(std::move(o.p)), r(o.r), c(o.c), cap(o.cap) { o.r = o.c = o.cap = 0; }
    DynStorage& operator=(const DynStorage& o) {
        if (this != &o) {
            resize_raw(o.r, o.c);
            if (r * c) std::memcpy(p.get(), o.p.get(), sizeof(S) * static_cast<std::size_t>(r * c));
        }
        return *this;
    }
    DynStorage& operator=(DynStorage&& o) noexcept {
        p = std::move(o.p);
        r = o.r;
        c = o.c;
        cap = o.cap;
        o.r = o.c = o.cap = 0;
        return *this;
    }
    S* ptr() { return p.get(); }
    const S* ptr() const { return p.get(); }
    /// Keeps the coefficients when the element count is unchanged (Eigen's resize); a new
    /// element count zero-fills (Eigen leaves it uninitialised: callers must not rely on it).
    bool resize_raw(Index nr, Index nc) {
        PSWARM_DENSE_CHECK(nr >= 0 && nc >= 0, "negative dimension");
        const Index n = nr * nc;
        const bool fresh = n != r * c || !p;
        if (n > cap || (n == 0 && cap)) {
            p.reset(n ? new S[static_cast<std::size_t>(n)] : nullptr);
            cap = n;
        }
        if (fresh && n) std::fill(p.get(), p.get() + n, S(0));
        r = nr;
        c = nc;
        return fresh;
    }
};
template <class S, int C>
struct Storage<S, Dynamic, C> : DynStorage<S> {
    Storage() { this->r = 0, this->c = C; }
    Index rows() const { return this->r; }
    Index cols() const { return C; }
};
template <class S, int R>
struct Storage<S, R, Dynamic> : DynStorage<S> {
    Storage() { this->r = R, this->c = 0; }
    Index rows() const { return R; }
    Index cols() const { return this->c; }
};
template <class S>
struct Storage<S, Dynamic, Dynamic> : DynStorage<S> {
    Index rows() const { return this->r; }
    Index cols() const { return this->c; }
};

// ---- the matrix product kernel: C (m x n) = A (m x k) * B (k x n), row-major
// contiguous rows (column stride 1) for A, B and C.  B is packed per column panel
// into 4-column tiles ([tile][k][4], zero-padded) so the micro-kernel streams it
// contiguously; register tiles of 4 rows x 4 columns (SSE2: eight 2-wide
// accumulators).  Every C coefficient is summed over k in order (p = 0..k-1).
inline void gemm_rowmajor(Index m, Index n, Index k, const double* A, Index lda, const double* B, Index ldb,
                          double* Cm, Index ldc) {
    constexpr Index NB = 128;  // columns per packed panel: k x 128 doubles (200 KB at k = 200)
    thread_local std::vector<double> pack;
    for (Index j0 = 0; j0 < n; j0 += NB) {
        const Index nb = std::min(NB, n - j0), nt = (nb + 3) / 4;
        pack.resize(static_cast<std::size_t>(nt * k * 4));
        double* pk = pack.data();
        for (Index t = 0; t < nt; ++t) {
            const Index c0 = j0 + 4 * t, w = std::min<Index>(4, n - c0);
            double* dst = pk + t * k * 4;
            for (Index p = 0; p < k; ++p) {
                const double* src = B + p * ldb + c0;
                for (Index q = 0; q < 4; ++q) dst[4 * p + q] = q < w ? src[q] : 0.0;
            }
        }
        Index i = 0;
        for (; i + 4 <= m; i += 4) {
            const double* a0 = A + (i + 0) * lda;
            const double* a1 = A + (i + 1) * lda;
            const double* a2 = A + (i + 2) * lda;
            const double* a3 = A + (i + 3) * lda;
            for (Index t = 0; t < nt; ++t) {
                const double* b = pk + t * k * 4;
                const Index c0 = j0 + 4 * t, w = std::min<Index>(4, n - c0);
                double acc[4][4];
#if defined(__SSE2__)
                if (w <= 2) {  // narrow last tile (e.g. the 6 columns of one trajectory): 4 x 2 kernel
                    __m128d c0v = _mm_setzero_pd(), c1v = _mm_setzero_pd(), c2v = _mm_setzero_pd(), c3v = _mm_setzero_pd();
                    for (Index p = 0; p < k; ++p, b += 4) {
                        const __m128d bv = _mm_load_pd(b);
                        c0v = _mm_add_pd(c0v, _mm_mul_pd(_mm_set1_pd(a0[p]), bv));
                        c1v = _mm_add_pd(c1v, _mm_mul_pd(_mm_set1_pd(a1[p]), bv));
                        c2v = _mm_add_pd(c2v, _mm_mul_pd(_mm_set1_pd(a2[p]), bv));
                        c3v = _mm_add_pd(c3v, _mm_mul_pd(_mm_set1_pd(a3[p]), bv));
                    }
                    _mm_storeu_pd(acc[0], c0v);
                    _mm_storeu_pd(acc[1], c1v);
                    _mm_storeu_pd(acc[2], c2v);
                    _mm_storeu_pd(acc[3], c3v);
                    for (Index r = 0; r < 4; ++r)
                        for (Index q = 0; q < w; ++q) Cm[(i + r) * ldc + c0 + q] = acc[r][q];
                    continue;
                }
                __m128d c00 = _mm_setzero_pd(), c01 = _mm_setzero_pd(), c10 = _mm_setzero_pd(), c11 = _mm_setzero_pd();
                __m128d c20 = _mm_setzero_pd(), c21 = _mm_setzero_pd(), c30 = _mm_setzero_pd(), c31 = _mm_setzero_pd();
                for (Index p = 0; p < k; ++p, b += 4) {
                    const __m128d b0 = _mm_load_pd(b), b1 = _mm_load_pd(b + 2);
                    __m128d x = _mm_set1_pd(a0[p]);
                    c00 = _mm_add_pd(c00, _mm_mul_pd(x, b0));
                    c01 = _mm_add_pd(c01, _mm_mul_pd(x, b1));
                    x = _mm_set1_pd(a1[p]);
                    c10 = _mm_add_pd(c10, _mm_mul_pd(x, b0));
                    c11 = _mm_add_pd(c11, _mm_mul_pd(x, b1));
                    x = _mm_set1_pd(a2[p]);
                    c20 = _mm_add_pd(c20, _mm_mul_pd(x, b0));
                    c21 = _mm_add_pd(c21, _mm_mul_pd(x, b1));
                    x = _mm_set1_pd(a3[p]);
                    c30 = _mm_add_pd(c30, _mm_mul_pd(x, b0));
                    c31 = _mm_add_pd(c31, _mm_mul_pd(x, b1));
                }
                _mm_storeu_pd(acc[0], c00);
                _mm_storeu_pd(acc[0] + 2, c01);
                _mm_storeu_pd(acc[1], c10);
                _mm_storeu_pd(acc[1] + 2, c11);
                _mm_storeu_pd(acc[2], c20);
                _mm_storeu_pd(acc[2] + 2, c21);
                _mm_storeu_pd(acc[3], c30);
                _mm_storeu_pd(acc[3] + 2, c31);
#else
                for (auto& r : acc)
                    for (double& v : r) v = 0.0;
                for (Index p = 0; p < k; ++p, b += 4)
                    for (Index q = 0; q < 4; ++q) {
                        acc[0][q] += a0[p] * b[q];
                        acc[1][q] += a1[p] * b[q];
                        acc[2][q] += a2[p] * b[q];
                        acc[3][q] += a3[p] * b[q];
                    }
#endif
                for (Index r = 0; r < 4; ++r)
                    for (Index q = 0; q < w; ++q) Cm[(i + r) * ldc + c0 + q] = acc[r][q];
            }
        }
        for (; i < m; ++i) {
            const double* a0 = A + i * lda;
            for (Index t = 0; t < nt; ++t) {
                const double* b = pk + t * k * 4;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                for (Index p = 0; p < k; ++p, b += 4)
                    for (Index q = 0; q < 4; ++q) acc[q] += a0[p] * b[q];
                const Index c0 = j0 + 4 * t, w = std::min<Index>(4, n - c0);
                for (Index q = 0; q < w; ++q) Cm[i * ldc + c0 + q] = acc[q];
            }
        }
    }
}
}  // namespace detail

template <class S, int R, int C, int Opt, int MR, int MC>
class Matrix : public DenseWritable<Matrix<S, R, C, Opt, MR, MC>> {
    using W = DenseWritable<Matrix>;

public:
    using Scalar = S;
    static constexpr bool IsRowMajor = (R == 1 && C != 1) ? true : (C == 1 && R != 1) ? false : bool(Opt & RowMajor);
    static constexpr bool IsFixed = R != Dynamic && C != Dynamic;
    static constexpr bool IsVec = R == 1 || C == 1;

    Matrix() = default;
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;

    /// dynamic vector: size; dynamic matrix: (rows, cols); fixed vector of 2..4: coefficients
    explicit Matrix(Index n) {
        static_assert(IsVec, "Matrix(n) needs a vector type");
        if constexpr (IsFixed) {
            PSWARM_DENSE_CHECK(n == R * C, "size mismatch");
        } else {
            resize(n);
            this->setZero();
        }
    }
    template <class I, class = std::enable_if_t<std::is_integral_v<I> && !IsFixed>>
    Matrix(I r, Index c) {
        resize(static_cast<Index>(r), c);
        this->setZero();
    }
    Matrix(S x, S y) requires(IsFixed && R * C == 2) { st_.a = {x, y}; }
    Matrix(S x, S y, S z) requires(IsFixed && R * C == 3) { st_.a = {x, y, z}; }
    Matrix(S x, S y, S z, S w) requires(IsFixed && R * C == 4) { st_.a = {x, y, z, w}; }
    Matrix(std::initializer_list<std::initializer_list<S>> rows) {
        const Index r = static_cast<Index>(rows.size());
        const Index c = r ? static_cast<Index>(rows.begin()->size()) : 0;
        resize(r, c);
        Index i = 0;
        for (const auto& rw : rows) {
            PSWARM_DENSE_CHECK(static_cast<Index>(rw.size()) == c, "ragged initializer list");
            Index j = 0;
            for (S v : rw) this->coeffRef(i, j++) = v;
            ++i;
        }
    }
    template <class O>
    Matrix(const DenseBase<O>& o) {
        resize_like(o);
        this->assign_from(o);
    }
    template <class O>
    Matrix& operator=(const DenseBase<O>& o) {
        if (static_cast<const void*>(o.data()) == static_cast<const void*>(this->data()) && o.data() != nullptr &&
            (o.rows() != this->rows() || o.cols() != this->cols() || o.rstride() != this->rstride())) {
            Matrix tmp(o);  // aliasing reshape (e.g. m = m.transpose())
            *this = std::move(tmp);
            return *this;
        }
        resize_like(o);
        this->assign_from(o);
        return *this;
    }

    void swap(Matrix& o) noexcept { std::swap(st_, o.st_); }

    // ---- storage
    Index rows_() const { return st_.rows(); }
    Index cols_() const { return st_.cols(); }
    Index rstride_() const { return IsRowMajor ? st_.cols() : 1; }
    Index cstride_() const { return IsRowMajor ? 1 : st_.rows(); }
    const S* cdata_() const { return st_.ptr(); }
    S* mdata_() { return st_.ptr(); }

    void resize(Index r, Index c) {
        if constexpr (IsFixed) {
            st_.resize(r, c);
        } else {
            PSWARM_DENSE_CHECK((R == Dynamic || r == R) && (C == Dynamic || c == C), "resize: fixed dimension changed");
            st_.resize_raw(r, c);
        }
    }
    void resize(Index n) {
        static_assert(IsVec, "resize(n) needs a vector type");
        if constexpr (R == 1)
            resize(1, n);
        else
            resize(n, 1);
    }
    void conservativeResize(Index r, Index c) {
        Matrix tmp(r, c);
        for (Index i = 0; i < std::min(r, rows_()); ++i)
            for (Index j = 0; j < std::min(c, cols_()); ++j) tmp(i, j) = (*this)(i, j);
        *this = std::move(tmp);
    }
    void conservativeResize(Index n) {
        if constexpr (R == 1)
            conservativeResize(1, n);
        else
            conservativeResize(n, 1);
    }
    using W::setZero;
    Matrix& setZero(Index n) {
        resize(n);
        return this->setConstant(S(0));
    }
    Matrix& setZero(Index r, Index c) {
        resize(r, c);
        return this->setConstant(S(0));
    }
    template <class O>
    void resize_like(const DenseBase<O>& o) {
        if constexpr (IsVec && !IsFixed) {
            if (o.is_vector()) {
                resize(o.size());
                return;
            }
        }
        if constexpr (IsFixed) {
            PSWARM_DENSE_CHECK(o.size() == R * C, "size mismatch assigning to a fixed-size matrix");
        } else {
            resize(o.rows(), o.cols());
        }
    }

    // ---- constructors of special matrices
    static Matrix Constant(Index r, Index c, S v) {
        Matrix m;
        m.resize(r, c);
        m.setConstant(v);
        return m;
    }
    static Matrix Constant(Index n, S v) {
        Matrix m;
        m.resize(n);
        m.setConstant(v);
        return m;
    }
    static Matrix Constant(S v) requires IsFixed {
        Matrix m;
        m.setConstant(v);
        return m;
    }
    static Matrix Zero(Index r, Index c) { return Constant(r, c, S(0)); }
    static Matrix Zero(Index n) { return Constant(n, S(0)); }
    static Matrix Zero() requires IsFixed { return Matrix(); }
    static Matrix Ones(Index r, Index c) { return Constant(r, c, S(1)); }
    static Matrix Ones(Index n) { return Constant(n, S(1)); }
    static Matrix Ones() requires IsFixed { return Constant(S(1)); }
    static Matrix Identity(Index r, Index c) {
        Matrix m = Zero(r, c);
        m.setIdentity();
        return m;
    }
    static Matrix Identity() requires IsFixed {
        Matrix m;
        m.setIdentity();
        return m;
    }
    static Matrix Unit(Index n, Index i) {
        Matrix m = Zero(n);
        m.coeffRef(i) = S(1);
        return m;
    }
    static Matrix Unit(Index i) requires IsFixed {
        Matrix m;
        m.coeffRef(i) = S(1);
        return m;
    }
    static Matrix UnitX() requires IsFixed { return Unit(0); }
    static Matrix UnitY() requires IsFixed { return Unit(1); }
    static Matrix UnitZ() requires IsFixed { return Unit(2); }
    static Matrix LinSpaced(Index n, S lo, S hi) {
        Matrix m;
        m.resize(n);
        for (Index k = 0; k < n; ++k)
            m.coeffRef(k) = (n == 1) ? hi : (k == n - 1 ? hi : lo + (hi - lo) * S(k) / S(n - 1));
        return m;
    }

    /// uninitialised construction for kernels that overwrite every coefficient
    static Matrix uninitialized(Index r, Index c) {
        Matrix m;
        m.resize(r, c);
        return m;
    }

private:
    detail::Storage<S, R, C> st_;
};

/// Map: a view over caller memory with the storage order of MatrixType.
template <class MatrixType>
class Map;
template <class S, int R, int C, int Opt, int MR, int MC>
class Map<Matrix<S, R, C, Opt, MR, MC>> : public View<S, R, C, false> {
    using M = Matrix<S, R, C, Opt, MR, MC>;
    using V = View<S, R, C, false>;

public:
    Map(S* p, Index n) : V(p, R == 1 ? 1 : n, R == 1 ? n : 1, R == 1 ? n : 1, 1) {
        static_assert(M::IsVec, "Map(p, n) needs a vector type");
    }
    Map(S* p, Index r, Index c) : V(p, r, c, M::IsRowMajor ? c : 1, M::IsRowMajor ? 1 : r) {}
    explicit Map(S* p) requires M::IsFixed : Map(p, R, C) {}
    using V::operator=;
};
template <class S, int R, int C, int Opt, int MR, int MC>
class Map<const Matrix<S, R, C, Opt, MR, MC>> : public View<S, R, C, true> {
    using M = Matrix<S, R, C, Opt, MR, MC>;
    using V = View<S, R, C, true>;

public:
    Map(const S* p, Index n) : V(p, R == 1 ? 1 : n, R == 1 ? n : 1, R == 1 ? n : 1, 1) {
        static_assert(M::IsVec, "Map(p, n) needs a vector type");
    }
    Map(const S* p, Index r, Index c) : V(p, r, c, M::IsRowMajor ? c : 1, M::IsRowMajor ? 1 : r) {}
    explicit Map(const S* p) requires M::IsFixed : Map(p, R, C) {}
};
template <class S, int R, int C, int Opt, int MR, int MC>
struct traits<Map<Matrix<S, R, C, Opt, MR, MC>>> : traits<View<S, R, C, false>> {};
template <class S, int R, int C, int Opt, int MR, int MC>
struct traits<Map<const Matrix<S, R, C, Opt, MR, MC>>> : traits<View<S, R, C, true>> {};

// ---------------------------------------------------------------------------
// Arithmetic (eager).
namespace detail {
template <class A, class B>
using BinaryPlain = Plain<typename traits<A>::Scalar, pick(traits<A>::Rows, traits<B>::Rows),
                          pick(traits<A>::Cols, traits<B>::Cols)>;

template <class A, class B, class F>
BinaryPlain<A, B> binary(const DenseBase<A>& a, const DenseBase<B>& b, F&& f) {
    using Out = BinaryPlain<A, B>;
    Out out(a);
    out.zip(b, [&](auto& x, auto y) { x = f(x, y); });
    return out;
}
}  // namespace detail

template <class Derived>
template <class O, class F>
typename DenseBase<Derived>::PlainObject DenseBase<Derived>::binaryExpr(const DenseBase<O>& o, F&& f) const {
    PlainObject out(derived());
    out.zip(o, [&](Scalar& x, Scalar y) { x = f(x, y); });
    return out;
}

template <class A, class B>
auto operator+(const DenseBase<A>& a, const DenseBase<B>& b) {
    return detail::binary(a, b, [](auto x, auto y) { return x + y; });
}
template <class A, class B>
auto operator-(const DenseBase<A>& a, const DenseBase<B>& b) {
    return detail::binary(a, b, [](auto x, auto y) { return x - y; });
}
template <class A>
typename DenseBase<A>::PlainObject operator-(const DenseBase<A>& a) {
    typename DenseBase<A>::PlainObject out(a);
    out.apply([](auto& x) { x = -x; });
    return out;
}
template <class A>
typename DenseBase<A>::PlainObject operator*(const DenseBase<A>& a, typename traits<A>::Scalar s) {
    typename DenseBase<A>::PlainObject out(a);
    out.apply([s](auto& x) { x = x * s; });
    return out;
}
template <class A>
typename DenseBase<A>::PlainObject operator*(typename traits<A>::Scalar s, const DenseBase<A>& a) {
    typename DenseBase<A>::PlainObject out(a);
    out.apply([s](auto& x) { x = s * x; });
    return out;
}
template <class A>
typename DenseBase<A>::PlainObject operator/(const DenseBase<A>& a, typename traits<A>::Scalar s) {
    typename DenseBase<A>::PlainObject out(a);
    out.apply([s](auto& x) { x = x / s; });
    return out;
}

/// Matrix product (A: r x k, B: k x c).
template <class A, class B>
auto operator*(const DenseBase<A>& a, const DenseBase<B>& b) {
    using S = typename traits<A>::Scalar;
    using Out = Plain<S, traits<A>::Rows, traits<B>::Cols>;
    PSWARM_DENSE_CHECK(a.cols() == b.rows(), "product: inner dimensions " + std::to_string(a.cols()) + " vs " +
                                                 std::to_string(b.rows()));
    const Index m = a.rows(), n = b.cols(), k = a.cols();
    Out out;
    if constexpr (Out::IsFixed) {
        out.setZero();
    } else {
        out.resize(m, n);
    }
    if constexpr (std::is_same_v<S, double>) {
        if (m * n * k >= 64 && a.cstride() == 1 && b.cstride() == 1 && (out.cstride() == 1 || n == 1)) {
            // row-major operands, output rows contiguous (a column-vector output has row stride 1)
            const Index ldc = (n == 1) ? 1 : out.rstride();
            detail::gemm_rowmajor(m, n, k, a.data(), a.rstride(), b.data(), b.rstride(), out.data(), ldc);
            return out;
        }
    }
    for (Index i = 0; i < m; ++i)
        for (Index j = 0; j < n; ++j) {
            S s = 0;
            for (Index p = 0; p < k; ++p) s += a.coeff(i, p) * b.coeff(p, j);
            out.coeffRef(i, j) = s;
        }
    return out;
}

/// Eigen's operator== on matrices: true when every coefficient compares equal.
template <class A, class B>
bool operator==(const DenseBase<A>& a, const DenseBase<B>& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j)
            if (!(a.coeff(i, j) == b.coeff(i, j))) return false;
    return true;
}
template <class A, class B>
bool operator!=(const DenseBase<A>& a, const DenseBase<B>& b) {
    return !(a == b);
}

template <class A>
std::ostream& operator<<(std::ostream& os, const DenseBase<A>& a) {
    for (Index i = 0; i < a.rows(); ++i) {
        for (Index j = 0; j < a.cols(); ++j) os << (j ? " " : "") << a.coeff(i, j);
        if (i + 1 < a.rows()) os << "\n";
    }
    return os;
}

// ---------------------------------------------------------------------------
// rowwise(): broadcast a row vector over every row.
template <class Derived>
class RowwiseProxy {
public:
    explicit RowwiseProxy(Derived& d) : d_(d) {}
    template <class O>
    Derived& operator=(const DenseBase<O>& r) {
        return each(r, [](auto& x, auto y) { x = y; });
    }
    template <class O>
    Derived& operator+=(const DenseBase<O>& r) {
        return each(r, [](auto& x, auto y) { x += y; });
    }
    template <class O>
    Derived& operator-=(const DenseBase<O>& r) {
        return each(r, [](auto& x, auto y) { x -= y; });
    }
    auto norm() const {
        Plain<typename traits<Derived>::Scalar, traits<Derived>::Rows, 1> out;
        out.resize(d_.rows(), 1);
        for (Index i = 0; i < d_.rows(); ++i) out.coeffRef(i) = d_.row(i).norm();
        return out;
    }
    auto maxCoeff() const {
        Plain<typename traits<Derived>::Scalar, traits<Derived>::Rows, 1> out;
        out.resize(d_.rows(), 1);
        for (Index i = 0; i < d_.rows(); ++i) out.coeffRef(i) = d_.row(i).maxCoeff();
        return out;
    }

private:
    template <class O, class F>
    Derived& each(const DenseBase<O>& r, F&& f) {
        PSWARM_DENSE_CHECK(r.is_vector() && r.size() == d_.cols(), "rowwise: vector length must equal cols");
        const Index rows = d_.rows(), cols = d_.cols();
        for (Index i = 0; i < rows; ++i)
            for (Index j = 0; j < cols; ++j) f(d_.coeffRef(i, j), r.coeff(j));
        return d_;
    }
    Derived& d_;
};

// ---------------------------------------------------------------------------
// array(): coefficient-wise view (comparisons, element-wise products, ...).
template <class S, int R, int C>
class ArrayPlain;
template <int R, int C>
class BoolArray {
public:
    BoolArray(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c)) {}
    void set(Index i, Index j, bool b) { v_[static_cast<std::size_t>(i * c_ + j)] = b ? 1 : 0; }
    bool all() const { return std::all_of(v_.begin(), v_.end(), [](char b) { return b != 0; }); }
    bool any() const { return std::any_of(v_.begin(), v_.end(), [](char b) { return b != 0; }); }
    Index count() const { return std::count_if(v_.begin(), v_.end(), [](char b) { return b != 0; }); }
    Index rows() const { return r_; }
    Index cols() const { return c_; }

private:
    Index r_, c_;
    std::vector<char> v_;
};

template <class Derived>
class ArrayView {
public:
    using Scalar = typename traits<Derived>::Scalar;
    static constexpr int R = traits<Derived>::Rows, C = traits<Derived>::Cols;
    using ArrayOut = ArrayPlain<Scalar, R, C>;
    explicit ArrayView(const DenseBase<Derived>& d) : d_(d.derived()) {}
    Index rows() const { return d_.rows(); }
    Index cols() const { return d_.cols(); }
    Scalar coeff(Index i, Index j) const { return d_.coeff(i, j); }
    const Derived& matrix() const { return d_; }
    template <class F>
    ArrayOut map(F&& f) const {
        ArrayOut out(rows(), cols());
        for (Index i = 0; i < rows(); ++i)
            for (Index j = 0; j < cols(); ++j) out.m.coeffRef(i, j) = f(coeff(i, j));
        return out;
    }
    ArrayOut abs() const {
        return map([](Scalar v) { return std::abs(v); });
    }
    ArrayOut square() const {
        return map([](Scalar v) { return v * v; });
    }
    ArrayOut sqrt() const {
        return map([](Scalar v) { return std::sqrt(v); });
    }
    Scalar sum() const { return d_.sum(); }
    Scalar maxCoeff() const { return d_.maxCoeff(); }
    Scalar minCoeff() const { return d_.minCoeff(); }
    bool allFinite() const { return d_.allFinite(); }

private:
    const Derived& d_;
};

template <class S, int R, int C>
class ArrayPlain {
public:
    ArrayPlain(Index r, Index c) { m.resize(r, c); }
    Index rows() const { return m.rows(); }
    Index cols() const { return m.cols(); }
    S coeff(Index i, Index j) const { return m.coeff(i, j); }
    const Plain<S, R, C>& matrix() const { return m; }
    S sum() const { return m.sum(); }
    S maxCoeff() const { return m.maxCoeff(); }
    S minCoeff() const { return m.minCoeff(); }
    ArrayPlain abs() const { return map([](S v) { return std::abs(v); }); }
    ArrayPlain square() const { return map([](S v) { return v * v; }); }
    ArrayPlain sqrt() const { return map([](S v) { return std::sqrt(v); }); }
    bool allFinite() const { return m.allFinite(); }
    template <class F>
    ArrayPlain map(F&& f) const {
        ArrayPlain out(rows(), cols());
        for (Index i = 0; i < rows(); ++i)
            for (Index j = 0; j < cols(); ++j) out.m.coeffRef(i, j) = f(coeff(i, j));
        return out;
    }
    Plain<S, R, C> m;
};

namespace detail {
template <class T>
struct is_array_like : std::false_type {};
template <class D>
struct is_array_like<ArrayView<D>> : std::true_type {};
template <class S, int R, int C>
struct is_array_like<ArrayPlain<S, R, C>> : std::true_type {};
template <class T>
inline constexpr bool is_array_v = is_array_like<std::decay_t<T>>::value;

template <class A, class B, class F>
auto array_zip(const A& a, const B& b, F&& f) {
    using S = decltype(a.coeff(0, 0));
    using Out = ArrayPlain<std::decay_t<S>, Dynamic, Dynamic>;
    PSWARM_DENSE_CHECK(a.rows() == b.rows() && a.cols() == b.cols(), "array shape mismatch");
    Out out(a.rows(), a.cols());
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j) out.m.coeffRef(i, j) = f(a.coeff(i, j), b.coeff(i, j));
    return out;
}
template <class A, class B, class F>
auto array_cmp(const A& a, const B& b, F&& f) {
    PSWARM_DENSE_CHECK(a.rows() == b.rows() && a.cols() == b.cols(), "array shape mismatch");
    BoolArray<Dynamic, Dynamic> out(a.rows(), a.cols());
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j) out.set(i, j, f(a.coeff(i, j), b.coeff(i, j)));
    return out;
}
template <class A, class F>
auto array_cmp_s(const A& a, double s, F&& f) {
    BoolArray<Dynamic, Dynamic> out(a.rows(), a.cols());
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j) out.set(i, j, f(a.coeff(i, j), s));
    return out;
}
}  // namespace detail

#define PSWARM_ARRAY_OP(op)                                                                                   \
    template <class A, class B, std::enable_if_t<detail::is_array_v<A> && detail::is_array_v<B>, int> = 0>   \
    auto operator op(const A& a, const B& b) {                                                                \
        return detail::array_zip(a, b, [](auto x, auto y) { return x op y; });                               \
    }                                                                                                         \
    template <class A, std::enable_if_t<detail::is_array_v<A>, int> = 0>                                       \
    auto operator op(const A& a, double s) {                                                                  \
        return a.map([s](auto x) { return x op s; });                                                         \
    }                                                                                                         \
    template <class A, std::enable_if_t<detail::is_array_v<A>, int> = 0>                                       \
    auto operator op(double s, const A& a) {                                                                  \
        return a.map([s](auto x) { return s op x; });                                                         \
    }
PSWARM_ARRAY_OP(+)
PSWARM_ARRAY_OP(-)
PSWARM_ARRAY_OP(*)
PSWARM_ARRAY_OP(/)
#undef PSWARM_ARRAY_OP

#define PSWARM_ARRAY_CMP(op)                                                                                  \
    template <class A, class B, std::enable_if_t<detail::is_array_v<A> && detail::is_array_v<B>, int> = 0>   \
    auto operator op(const A& a, const B& b) {                                                                \
        return detail::array_cmp(a, b, [](auto x, auto y) { return x op y; });                               \
    }                                                                                                         \
    template <class A, std::enable_if_t<detail::is_array_v<A>, int> = 0>                                       \
    auto operator op(const A& a, double s) {                                                                  \
        return detail::array_cmp_s(a, s, [](auto x, auto y) { return x op y; });                             \
    }
PSWARM_ARRAY_CMP(==)
PSWARM_ARRAY_CMP(!=)
PSWARM_ARRAY_CMP(<)
PSWARM_ARRAY_CMP(<=)
PSWARM_ARRAY_CMP(>)
PSWARM_ARRAY_CMP(>=)
#undef PSWARM_ARRAY_CMP

// ---------------------------------------------------------------------------
// Common aliases (Eigen names).
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Matrix3d = Matrix<double, 3, 3>;
using RowVector3d = Matrix<double, 1, 3>;

}  // namespace pswarm::dense
