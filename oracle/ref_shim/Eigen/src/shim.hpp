// Eigen-subset shim — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// The reference (proj/, CMakeLists.txt:29) needs Eigen 3, which is not
// installed in this image and has no pinned version.  This header restates
// the part of Eigen 3.x's dense API and arithmetic that the reference's
// sources and tests use, so that oracle/ref_build.py can compile
// /root/reference/proj/src/*.cpp and proj/tests/*.cpp UNMODIFIED into
// oracle/_ref/ (the reference run as the parity anchor).  Nothing under
// paper_2208_04726_b200/ includes it.
//
// Model: every object is strided storage.  Matrix<> owns column-major
// storage; blocks / rows / cols / diagonals / transposes are strided views of
// it; every arithmetic expression is evaluated eagerly into a Matrix<> whose
// compile-time shape follows Eigen's rules.  Scalar arithmetic follows
// Eigen's unvectorised formulas (sequential reductions, the quaternion
// product and rotation formulas of Quaternion.h, LDLT's symmetric pivoting of
// LDLT.h); vectorised Eigen builds may round differently in the last ulp.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <string>
#include <cstddef>
#include <initializer_list>
#include <iostream>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum StorageOptions { ColMajor = 0, RowMajor = 0x1, AutoAlign = 0, DontAlign = 0x2 };
enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20 };

template <class S, int R, int C, int O = 0, int MR = R, int MC = C>
class Matrix;
template <class S, int R, int C>
class View;
template <class S, int R, int C>
class ArrayView;
template <class S, int N>
class DiagonalWrapper;
template <class M>
class LDLT;
template <class M>
class FullPivLU;
template <class M>
class ColPivHouseholderQR;

namespace internal {
constexpr int prod_dim(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : a * b; }
constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }
constexpr int min_dim(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : (a < b ? a : b); }
[[noreturn]] inline void fail(const char* what) { throw std::logic_error(std::string("Eigen shim: ") + what); }
}  // namespace internal

// Strided element window: element (i, j) lives at p[i * rs + j * cs].
template <class S>
struct Desc {
    S* p;
    Index r, c, rs, cs;
    S& at(Index i, Index j) const { return p[i * rs + j * cs]; }
};

// ---------------------------------------------------------------------------
// MBase: the dense-matrix interface shared by Matrix and View (CRTP)
// ---------------------------------------------------------------------------
template <class D, class S, int R, int C>
class MBase {
  public:
    using Scalar = S;
    using RealScalar = S;
    static constexpr int RowsAtCompileTime = R;
    static constexpr int ColsAtCompileTime = C;
    static constexpr int SizeAtCompileTime = internal::prod_dim(R, C);
    static constexpr bool IsVectorAtCompileTime = (R == 1 || C == 1);
    using PlainObject = Matrix<S, R, C>;

    const D& derived() const { return static_cast<const D&>(*this); }
    D& derived() { return static_cast<D&>(*this); }
    Desc<S> desc() const { return derived().desc_(); }

    Index rows() const { return desc().r; }
    Index cols() const { return desc().c; }
    Index size() const { return rows() * cols(); }

    S& coeffRef(Index i, Index j) const { return desc().at(i, j); }
    S coeff(Index i, Index j) const { return desc().at(i, j); }
    S& operator()(Index i, Index j) const { return desc().at(i, j); }
    // linear access: vectors by position, matrices column-major
    S& lin(Index k) const {
        const Desc<S> d = desc();
        if (d.c == 1) return d.at(k, 0);
        if (d.r == 1) return d.at(0, k);
        return d.at(k % d.r, k / d.r);
    }
    S& operator()(Index k) const { return lin(k); }
    S& operator[](Index k) const { return lin(k); }
    S& coeffRef(Index k) const { return lin(k); }
    S coeff(Index k) const { return lin(k); }
    S& x() const { return lin(0); }
    S& y() const { return lin(1); }
    S& z() const { return lin(2); }
    S& w() const { return lin(3); }
    S value() const {
        if (size() != 1) internal::fail("value() of a non-1x1 matrix");
        return lin(0);
    }

    // ---- views ----
    template <int BR, int BC>
    View<S, BR, BC> block(Index i, Index j) const {
        const Desc<S> d = desc();
        return View<S, BR, BC>(Desc<S>{d.p + i * d.rs + j * d.cs, BR, BC, d.rs, d.cs});
    }
    View<S, Dynamic, Dynamic> block(Index i, Index j, Index nr, Index nc) const {
        const Desc<S> d = desc();
        return View<S, Dynamic, Dynamic>(Desc<S>{d.p + i * d.rs + j * d.cs, nr, nc, d.rs, d.cs});
    }
    View<S, Dynamic, Dynamic> topLeftCorner(Index nr, Index nc) const { return block(0, 0, nr, nc); }
    View<S, Dynamic, Dynamic> topRightCorner(Index nr, Index nc) const { return block(0, cols() - nc, nr, nc); }
    View<S, Dynamic, Dynamic> bottomLeftCorner(Index nr, Index nc) const { return block(rows() - nr, 0, nr, nc); }
    View<S, Dynamic, Dynamic> bottomRightCorner(Index nr, Index nc) const {
        return block(rows() - nr, cols() - nc, nr, nc);
    }
    template <int NR, int NC>
    View<S, NR, NC> topLeftCorner() const { return block<NR, NC>(0, 0); }
    template <int NR, int NC>
    View<S, NR, NC> topRightCorner() const { return block<NR, NC>(0, cols() - NC); }
    template <int NR, int NC>
    View<S, NR, NC> bottomLeftCorner() const { return block<NR, NC>(rows() - NR, 0); }
    template <int NR, int NC>
    View<S, NR, NC> bottomRightCorner() const { return block<NR, NC>(rows() - NR, cols() - NC); }
    template <int N>
    View<S, R, N> leftCols() const { return sub<R, N>(0, 0, rows(), N); }
    template <int N>
    View<S, R, N> rightCols() const { return sub<R, N>(0, cols() - N, rows(), N); }
    template <int N>
    View<S, N, C> topRows() const { return sub<N, C>(0, 0, N, cols()); }
    template <int N>
    View<S, N, C> bottomRows() const { return sub<N, C>(rows() - N, 0, N, cols()); }
    View<S, R, Dynamic> leftCols(Index n) const { return sub<R, Dynamic>(0, 0, rows(), n); }
    View<S, R, Dynamic> rightCols(Index n) const { return sub<R, Dynamic>(0, cols() - n, rows(), n); }
    View<S, R, Dynamic> middleCols(Index j, Index n) const { return sub<R, Dynamic>(0, j, rows(), n); }
    View<S, Dynamic, C> topRows(Index n) const { return sub<Dynamic, C>(0, 0, n, cols()); }
    View<S, Dynamic, C> bottomRows(Index n) const { return sub<Dynamic, C>(rows() - n, 0, n, cols()); }
    View<S, Dynamic, C> middleRows(Index i, Index n) const { return sub<Dynamic, C>(i, 0, n, cols()); }
    View<S, R, 1> col(Index j) const { return sub<R, 1>(0, j, rows(), 1); }
    View<S, 1, C> row(Index i) const { return sub<1, C>(i, 0, 1, cols()); }
    // vector segments (column or row vectors)
    template <int N>
    auto head() const { return seg<N>(0, N); }
    template <int N>
    auto tail() const { return seg<N>(size() - N, N); }
    template <int N>
    auto segment(Index o) const { return seg<N>(o, N); }
    auto head(Index n) const { return seg<Dynamic>(0, n); }
    auto tail(Index n) const { return seg<Dynamic>(size() - n, n); }
    auto segment(Index o, Index n) const { return seg<Dynamic>(o, n); }
    View<S, internal::min_dim(R, C), 1> diagonal() const {
        const Desc<S> d = desc();
        return View<S, internal::min_dim(R, C), 1>(Desc<S>{d.p, std::min(d.r, d.c), 1, d.rs + d.cs, 0});
    }
    View<S, C, R> transpose() const {
        const Desc<S> d = desc();
        return View<S, C, R>(Desc<S>{d.p, d.c, d.r, d.cs, d.rs});
    }
    View<S, C, R> adjoint() const { return transpose(); }
    ArrayView<S, R, C> array() const { return ArrayView<S, R, C>(desc()); }
    const D& matrix() const { return derived(); }
    View<S, R, C> real() const { return View<S, R, C>(desc()); }
    PlainObject eval() const { return PlainObject(*this); }
    S* data() const { return desc().p; }

    // ---- assignment helpers (through the view) ----
    template <class E, int R2, int C2>
    void assign_from(const MBase<E, S, R2, C2>& o) const {
        if (o.rows() != rows() || o.cols() != cols()) internal::fail("size mismatch in assignment");
        const Matrix<S, R2, C2> tmp(o);  // evaluate first: no aliasing surprises
        const Desc<S> d = desc();
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) d.at(i, j) = tmp.coeff(i, j);
    }
    template <class F>
    void apply(F f) const {
        const Desc<S> d = desc();
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) f(d.at(i, j));
    }
    template <class E, int R2, int C2>
    D& operator+=(const MBase<E, S, R2, C2>& o) {
        check_same(o);
        const Matrix<S, R2, C2> t(o);
        const Desc<S> d = desc();
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) d.at(i, j) += t.coeff(i, j);
        return derived();
    }
    template <class E, int R2, int C2>
    D& operator-=(const MBase<E, S, R2, C2>& o) {
        check_same(o);
        const Matrix<S, R2, C2> t(o);
        const Desc<S> d = desc();
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) d.at(i, j) -= t.coeff(i, j);
        return derived();
    }
    D& operator*=(S s) {
        apply([s](S& v) { v *= s; });
        return derived();
    }
    D& operator/=(S s) {
        apply([s](S& v) { v /= s; });
        return derived();
    }
    template <class E, int R2, int C2>
    D& operator*=(const MBase<E, S, R2, C2>& o) {
        derived() = derived() * o;
        return derived();
    }
    D& setZero() {
        apply([](S& v) { v = S(0); });
        return derived();
    }
    D& setOnes() {
        apply([](S& v) { v = S(1); });
        return derived();
    }
    D& setConstant(S s) {
        apply([s](S& v) { v = s; });
        return derived();
    }
    D& fill(S s) { return setConstant(s); }
    D& setIdentity() {
        const Desc<S> d = desc();
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) d.at(i, j) = (i == j) ? S(1) : S(0);
        return derived();
    }
    template <class E, int R2, int C2>
    void swap(const MBase<E, S, R2, C2>& o) const {
        check_same(o);
        const Desc<S> a = desc(), b = o.desc();
        for (Index j = 0; j < a.c; ++j)
            for (Index i = 0; i < a.r; ++i) std::swap(a.at(i, j), b.at(i, j));
    }
    void normalize() {
        const S n = squaredNorm();
        if (n > S(0)) derived() /= std::sqrt(n);
    }

    // ---- reductions ----
    S sum() const {
        const Desc<S> d = desc();
        if (d.r * d.c == 0) return S(0);
        S s = lin(0);
        for (Index k = 1; k < d.r * d.c; ++k) s += lin(k);
        return s;
    }
    S mean() const { return sum() / S(size()); }
    S trace() const { return diagonal().sum(); }
    S squaredNorm() const {
        const Index n = size();
        if (n == 0) return S(0);
        S s = lin(0) * lin(0);
        for (Index k = 1; k < n; ++k) s += lin(k) * lin(k);
        return s;
    }
    S norm() const { return std::sqrt(squaredNorm()); }
    S stableNorm() const { return norm(); }
    template <class E, int R2, int C2>
    S dot(const MBase<E, S, R2, C2>& o) const {
        if (o.size() != size()) internal::fail("dot size mismatch");
        if (size() == 0) return S(0);
        S s = lin(0) * o.lin(0);
        for (Index k = 1; k < size(); ++k) s += lin(k) * o.lin(k);
        return s;
    }
    S maxCoeff() const { return extreme(true, nullptr, nullptr); }
    S minCoeff() const { return extreme(false, nullptr, nullptr); }
    template <class I>
    S maxCoeff(I* idx) const {
        Index i, j;
        const S v = extreme(true, &i, &j);
        *idx = static_cast<I>(cols() == 1 ? i : (rows() == 1 ? j : i + j * rows()));
        return v;
    }
    template <class I>
    S minCoeff(I* idx) const {
        Index i, j;
        const S v = extreme(false, &i, &j);
        *idx = static_cast<I>(cols() == 1 ? i : (rows() == 1 ? j : i + j * rows()));
        return v;
    }
    template <class I>
    S maxCoeff(I* ri, I* ci) const {
        Index i, j;
        const S v = extreme(true, &i, &j);
        *ri = static_cast<I>(i);
        *ci = static_cast<I>(j);
        return v;
    }
    bool allFinite() const {
        bool ok = true;
        apply([&ok](S& v) { ok = ok && std::isfinite(v); });
        return ok;
    }
    bool hasNaN() const {
        bool nan = false;
        apply([&nan](S& v) { nan = nan || std::isnan(v); });
        return nan;
    }
    // Eigen's isMuchSmallerThan(x, 1, prec): |x| <= prec
    bool isZero(S prec = S(1e-12)) const {
        bool z = true;
        apply([&](S& v) { z = z && std::abs(v) <= prec; });
        return z;
    }
    bool isApprox(const PlainObject& o, S prec = S(1e-12)) const {
        const PlainObject diff = PlainObject(*this) - o;
        return diff.squaredNorm() <= prec * prec * std::min(squaredNorm(), o.squaredNorm());
    }

    // ---- coefficient-wise ----
    PlainObject cwiseAbs() const { return map([](S v) { return std::abs(v); }); }
    PlainObject cwiseAbs2() const { return map([](S v) { return v * v; }); }
    PlainObject cwiseInverse() const { return map([](S v) { return S(1) / v; }); }
    PlainObject cwiseSqrt() const { return map([](S v) { return std::sqrt(v); }); }
    template <class E, int R2, int C2>
    PlainObject cwiseProduct(const MBase<E, S, R2, C2>& o) const {
        return zip(o, [](S a, S b) { return a * b; });
    }
    template <class E, int R2, int C2>
    PlainObject cwiseQuotient(const MBase<E, S, R2, C2>& o) const {
        return zip(o, [](S a, S b) { return a / b; });
    }
    template <class E, int R2, int C2>
    PlainObject cwiseMax(const MBase<E, S, R2, C2>& o) const {
        return zip(o, [](S a, S b) { return a < b ? b : a; });
    }
    template <class E, int R2, int C2>
    PlainObject cwiseMin(const MBase<E, S, R2, C2>& o) const {
        return zip(o, [](S a, S b) { return b < a ? b : a; });
    }
    PlainObject normalized() const {
        const S n = squaredNorm();
        PlainObject out(*this);
        if (n > S(0)) out /= std::sqrt(n);
        return out;
    }
    DiagonalWrapper<S, (R == 1 ? C : R)> asDiagonal() const { return DiagonalWrapper<S, (R == 1 ? C : R)>(*this); }
    Matrix<S, 3, 1> cross(const Matrix<S, 3, 1>& b) const {
        return Matrix<S, 3, 1>(y() * b.z() - z() * b.y(), z() * b.x() - x() * b.z(), x() * b.y() - y() * b.x());
    }

    // ---- solvers ----
    LDLT<Matrix<S, R, C>> ldlt() const;
    FullPivLU<Matrix<S, R, C>> fullPivLu() const;
    ColPivHouseholderQR<Matrix<S, R, C>> colPivHouseholderQr() const;
    PlainObject inverse() const;
    S determinant() const;

    template <class F>
    PlainObject map(F f) const {
        PlainObject out(*this);
        out.apply([&f](S& v) { v = f(v); });
        return out;
    }
    template <class E, int R2, int C2, class F>
    PlainObject zip(const MBase<E, S, R2, C2>& o, F f) const {
        check_same(o);
        PlainObject out(*this);
        const Desc<S> a = out.desc(), b = o.desc();
        for (Index j = 0; j < a.c; ++j)
            for (Index i = 0; i < a.r; ++i) a.at(i, j) = f(a.at(i, j), b.at(i, j));
        return out;
    }
    template <class E, int R2, int C2>
    void check_same(const MBase<E, S, R2, C2>& o) const {
        if (o.rows() != rows() || o.cols() != cols()) internal::fail("operand size mismatch");
    }

  private:
    template <int NR, int NC>
    View<S, NR, NC> sub(Index i, Index j, Index nr, Index nc) const {
        const Desc<S> d = desc();
        return View<S, NR, NC>(Desc<S>{d.p + i * d.rs + j * d.cs, nr, nc, d.rs, d.cs});
    }
    template <int N>
    auto seg(Index o, Index n) const {
        const Desc<S> d = desc();
        if constexpr (R == 1) {
            return View<S, 1, N>(Desc<S>{d.p + o * d.cs, 1, n, d.rs, d.cs});
        } else {
            if (d.c != 1) internal::fail("segment of a non-vector");
            return View<S, N, 1>(Desc<S>{d.p + o * d.rs, n, 1, d.rs, d.cs});
        }
    }
    S extreme(bool want_max, Index* ri, Index* ci) const {
        const Desc<S> d = desc();
        if (d.r * d.c == 0) internal::fail("maxCoeff/minCoeff of an empty matrix");
        S best = d.at(0, 0);
        Index bi = 0, bj = 0;
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) {
                const S v = d.at(i, j);
                if (want_max ? (v > best) : (v < best)) {  // strict: the first extreme wins
                    best = v;
                    bi = i;
                    bj = j;
                }
            }
        if (ri) *ri = bi;
        if (ci) *ci = bj;
        return best;
    }
};

// ---------------------------------------------------------------------------
// comma initializer: fills row by row, blocks advance by their width/height
// ---------------------------------------------------------------------------
template <class S>
class CommaInit {
  public:
    explicit CommaInit(Desc<S> d) : d_(d) {}
    CommaInit(const CommaInit&) = delete;
    CommaInit(CommaInit&& o) noexcept : d_(o.d_), row_(o.row_), col_(o.col_), h_(o.h_) { o.moved_ = true; }
    ~CommaInit() {
        if (!moved_ && d_.r * d_.c > 0 && !(row_ + h_ == d_.r && col_ == d_.c)) {
            std::cerr << "Eigen shim: too few coefficients in comma initializer\n";
            std::abort();
        }
    }
    CommaInit& push(S v) {
        advance(1);
        d_.at(row_, col_) = v;
        col_ += 1;
        return *this;
    }
    template <class E, int R2, int C2>
    CommaInit& push(const MBase<E, S, R2, C2>& m) {
        if (m.size() == 0) return *this;
        advance(m.rows());
        if (col_ + m.cols() > d_.c || row_ + m.rows() > d_.r) internal::fail("comma initializer overflow");
        for (Index j = 0; j < m.cols(); ++j)
            for (Index i = 0; i < m.rows(); ++i) d_.at(row_ + i, col_ + j) = m.coeff(i, j);
        col_ += m.cols();
        return *this;
    }
    CommaInit& operator,(S v) { return push(v); }
    template <class E, int R2, int C2>
    CommaInit& operator,(const MBase<E, S, R2, C2>& m) {
        return push(m);
    }

  private:
    void advance(Index h) {
        if (col_ == d_.c) {  // row band full: next band
            row_ += h_;
            col_ = 0;
            h_ = h;
        } else if (col_ == 0) {
            h_ = h;
        } else if (h != h_) {
            internal::fail("inconsistent block heights in comma initializer");
        }
        if (row_ >= d_.r) internal::fail("comma initializer overflow");
    }
    Desc<S> d_;
    Index row_ = 0, col_ = 0, h_ = 1;
    bool moved_ = false;
};

// ---------------------------------------------------------------------------
// View: a strided window into some storage
// ---------------------------------------------------------------------------
template <class S, int R, int C>
class View : public MBase<View<S, R, C>, S, R, C> {
  public:
    using Base = MBase<View<S, R, C>, S, R, C>;
    explicit View(Desc<S> d) : d_(d) {}
    View(const View&) = default;
    Desc<S> desc_() const { return d_; }
    // assignment writes THROUGH the view
    View& operator=(const View& o) {
        this->assign_from(o);
        return *this;
    }
    template <class E, int R2, int C2>
    View& operator=(const MBase<E, S, R2, C2>& o) {
        this->assign_from(o);
        return *this;
    }
    template <int N>
    View& operator=(const DiagonalWrapper<S, N>& dw) {
        this->assign_from(Matrix<S, N, N>(dw));
        return *this;
    }
    CommaInit<S> operator<<(S v) {
        CommaInit<S> ci(d_);
        ci.push(v);
        return ci;
    }
    template <class E, int R2, int C2>
    CommaInit<S> operator<<(const MBase<E, S, R2, C2>& m) {
        CommaInit<S> ci(d_);
        ci.push(m);
        return ci;
    }
    using Base::operator+=;
    using Base::operator-=;
    using Base::operator*=;

  private:
    Desc<S> d_;
};

// ---------------------------------------------------------------------------
// Matrix: owning, column-major
// ---------------------------------------------------------------------------
template <class S, int R, int C, int O, int MR, int MC>
class Matrix : public MBase<Matrix<S, R, C, O, MR, MC>, S, R, C> {
    static constexpr bool kFixed = (R != Dynamic && C != Dynamic);
    using Store = std::conditional_t<kFixed, std::array<S, (kFixed ? R * C : 1)>, std::vector<S>>;

  public:
    using Base = MBase<Matrix, S, R, C>;
    Matrix() {
        if constexpr (kFixed) {
            v_.fill(S(0));
        } else {
            r_ = (R == Dynamic) ? 0 : R;
            c_ = (C == Dynamic) ? 0 : C;
        }
    }
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;

    // one argument: a size for dynamic vectors, else the single coefficient
    template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
    explicit Matrix(T n) {
        if constexpr (!kFixed) {
            if constexpr (R == 1) resize(1, static_cast<Index>(n));
            else resize(static_cast<Index>(n), 1);
        } else {
            static_assert(R * C == 1 || !kFixed, "scalar constructor of a non-1x1 fixed matrix");
            v_[0] = static_cast<S>(n);
        }
    }
    // two arguments: coefficients of a fixed 2-vector, else the sizes
    template <class T0, class T1,
              std::enable_if_t<std::is_arithmetic_v<T0> && std::is_arithmetic_v<T1>, int> = 0>
    Matrix(T0 a, T1 b) {
        if constexpr (kFixed && R * C == 2) {
            v_[0] = static_cast<S>(a);
            v_[1] = static_cast<S>(b);
        } else if constexpr (!kFixed) {
            resize(static_cast<Index>(a), static_cast<Index>(b));
        } else {
            static_assert(R * C == 2, "two-coefficient constructor needs a 2-vector");
        }
    }
    Matrix(S a, S b, S c) {
        init_size(3);
        v_[0] = a, v_[1] = b, v_[2] = c;
    }
    Matrix(S a, S b, S c, S d) {
        init_size(4);
        v_[0] = a, v_[1] = b, v_[2] = c, v_[3] = d;
    }
    template <class E, int R2, int C2>
    Matrix(const MBase<E, S, R2, C2>& o) {  // NOLINT: implicit like Eigen's expression conversion
        resize(o.rows(), o.cols());
        const Desc<S> s = o.desc();
        for (Index j = 0; j < s.c; ++j)
            for (Index i = 0; i < s.r; ++i) v_[i + j * rows_()] = s.at(i, j);
    }
    template <int N>
    Matrix(const DiagonalWrapper<S, N>& dw) {  // NOLINT
        const Index n = dw.diagonal().size();
        resize(n, n);
        this->setZero();
        for (Index k = 0; k < n; ++k) v_[k + k * n] = dw.diagonal()(k);
    }
    template <class E, int R2, int C2>
    Matrix& operator=(const MBase<E, S, R2, C2>& o) {
        Matrix tmp(o);
        *this = std::move(tmp);
        return *this;
    }
    template <int N>
    Matrix& operator=(const DiagonalWrapper<S, N>& dw) {
        *this = Matrix(dw);
        return *this;
    }

    Desc<S> desc_() const {
        return Desc<S>{const_cast<S*>(v_.data()), rows_(), cols_(), 1, rows_()};
    }
    void resize(Index nr, Index nc) {
        if constexpr (kFixed) {
            if (nr != R || nc != C) internal::fail("resizing a fixed-size matrix");
        } else {
            if ((R != Dynamic && nr != R) || (C != Dynamic && nc != C)) internal::fail("resize against a fixed dimension");
            r_ = nr;
            c_ = nc;
            v_.assign(static_cast<size_t>(nr * nc), S(0));
        }
    }
    void resize(Index n) {
        if constexpr (R == 1) resize(1, n);
        else resize(n, 1);
    }
    void conservativeResize(Index n) {
        Matrix old = *this;
        resize(n);
        for (Index k = 0; k < std::min(n, old.size()); ++k) v_[k] = old.v_[k];
    }

    CommaInit<S> operator<<(S v) {
        CommaInit<S> ci(this->desc());
        ci.push(v);
        return ci;
    }
    template <class E, int R2, int C2>
    CommaInit<S> operator<<(const MBase<E, S, R2, C2>& m) {
        CommaInit<S> ci(this->desc());
        ci.push(m);
        return ci;
    }

    // ---- static constructors ----
    static Matrix Zero() { return Constant(S(0)); }
    static Matrix Zero(Index n) { return Constant(n, S(0)); }
    static Matrix Zero(Index nr, Index nc) { return Constant(nr, nc, S(0)); }
    static Matrix Ones() { return Constant(S(1)); }
    static Matrix Ones(Index n) { return Constant(n, S(1)); }
    static Matrix Ones(Index nr, Index nc) { return Constant(nr, nc, S(1)); }
    static Matrix Constant(S v) {
        Matrix m;
        m.setConstant(v);
        return m;
    }
    static Matrix Constant(Index n, S v) {
        Matrix m;
        m.resize(n);
        m.setConstant(v);
        return m;
    }
    static Matrix Constant(Index nr, Index nc, S v) {
        Matrix m;
        m.resize(nr, nc);
        m.setConstant(v);
        return m;
    }
    static Matrix Identity() {
        Matrix m;
        m.setIdentity();
        return m;
    }
    static Matrix Identity(Index nr, Index nc) {
        Matrix m;
        m.resize(nr, nc);
        m.setIdentity();
        return m;
    }
    static Matrix Unit(Index i) {
        Matrix m = Zero();
        m(i) = S(1);
        return m;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }
    static Matrix UnitW() { return Unit(3); }

    using Base::operator+=;
    using Base::operator-=;
    using Base::operator*=;

  private:
    Index rows_() const {
        if constexpr (kFixed) return R;
        else return r_;
    }
    Index cols_() const {
        if constexpr (kFixed) return C;
        else return c_;
    }
    void init_size(Index n) {
        if constexpr (kFixed) {
            if (R * C != n) internal::fail("coefficient count does not match the fixed size");
        } else {
            resize(n);
        }
    }
    Store v_{};
    Index r_ = 0, c_ = 0;
};

// ---------------------------------------------------------------------------
// Arrays (.array()): coefficient-wise semantics over the same storage
// ---------------------------------------------------------------------------
template <class S, int R, int C>
class ArrayView {
  public:
    explicit ArrayView(Desc<S> d) : d_(d) {}
    Index size() const { return d_.r * d_.c; }
    template <class F>
    void apply(F f) const {
        for (Index j = 0; j < d_.c; ++j)
            for (Index i = 0; i < d_.r; ++i) f(d_.at(i, j));
    }
    ArrayView& operator+=(S s) {
        apply([s](S& v) { v += s; });
        return *this;
    }
    ArrayView& operator-=(S s) {
        apply([s](S& v) { v -= s; });
        return *this;
    }
    ArrayView& operator*=(S s) {
        apply([s](S& v) { v *= s; });
        return *this;
    }
    ArrayView& operator/=(S s) {
        apply([s](S& v) { v /= s; });
        return *this;
    }
    Matrix<S, R, C> matrix() const { return Matrix<S, R, C>(View<S, R, C>(d_)); }
    S sum() const { return View<S, R, C>(d_).sum(); }
    S maxCoeff() const { return View<S, R, C>(d_).maxCoeff(); }
    S minCoeff() const { return View<S, R, C>(d_).minCoeff(); }
    ArrayView<S, R, C> abs() const = delete;  // not needed by the reference

    struct BoolArray {
        std::vector<bool> b;
        bool any() const { return std::any_of(b.begin(), b.end(), [](bool v) { return v; }); }
        bool all() const { return std::all_of(b.begin(), b.end(), [](bool v) { return v; }); }
        Index count() const { return std::count(b.begin(), b.end(), true); }
    };
    template <class F>
    BoolArray cmp(F f) const {
        BoolArray out;
        apply([&](S& v) { out.b.push_back(f(v)); });
        return out;
    }
    BoolArray operator<=(S s) const { return cmp([s](S v) { return v <= s; }); }
    BoolArray operator<(S s) const { return cmp([s](S v) { return v < s; }); }
    BoolArray operator>=(S s) const { return cmp([s](S v) { return v >= s; }); }
    BoolArray operator>(S s) const { return cmp([s](S v) { return v > s; }); }
    BoolArray operator==(S s) const { return cmp([s](S v) { return v == s; }); }
    BoolArray operator!=(S s) const { return cmp([s](S v) { return v != s; }); }

  private:
    Desc<S> d_;
};

// ---------------------------------------------------------------------------
// DiagonalWrapper (asDiagonal): scales rows / columns in products
// ---------------------------------------------------------------------------
template <class S, int N>
class DiagonalWrapper {
  public:
    template <class E, int R2, int C2>
    explicit DiagonalWrapper(const MBase<E, S, R2, C2>& v) : d_(Matrix<S, N, 1>::Zero(v.size())) {
        for (Index k = 0; k < v.size(); ++k) d_(k) = v.lin(k);
    }
    const Matrix<S, N, 1>& diagonal() const { return d_; }
    Index rows() const { return d_.size(); }
    Index cols() const { return d_.size(); }

  private:
    Matrix<S, N, 1> d_;
};

// ---------------------------------------------------------------------------
// arithmetic operators (eager)
// ---------------------------------------------------------------------------
template <class A, class B, class S, int R1, int C1, int R2, int C2>
Matrix<S, internal::pick(R1, R2), internal::pick(C1, C2)> operator+(const MBase<A, S, R1, C1>& a,
                                                                     const MBase<B, S, R2, C2>& b) {
    Matrix<S, internal::pick(R1, R2), internal::pick(C1, C2)> out(a);
    out += b;
    return out;
}
template <class A, class B, class S, int R1, int C1, int R2, int C2>
Matrix<S, internal::pick(R1, R2), internal::pick(C1, C2)> operator-(const MBase<A, S, R1, C1>& a,
                                                                     const MBase<B, S, R2, C2>& b) {
    Matrix<S, internal::pick(R1, R2), internal::pick(C1, C2)> out(a);
    out -= b;
    return out;
}
template <class A, class S, int R, int C>
Matrix<S, R, C> operator-(const MBase<A, S, R, C>& a) {
    return a.map([](S v) { return -v; });
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator*(const MBase<A, S, R, C>& a, T s) {
    const S k = static_cast<S>(s);
    return a.map([k](S v) { return v * k; });
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator*(T s, const MBase<A, S, R, C>& a) {
    const S k = static_cast<S>(s);
    return a.map([k](S v) { return k * v; });
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator/(const MBase<A, S, R, C>& a, T s) {
    const S k = static_cast<S>(s);
    return a.map([k](S v) { return v / k; });
}
// matrix product: every coefficient a sequential inner sum (Eigen's lazy
// coefficient-based product; its blocked GEMM may associate differently)
template <class A, class B, class S, int R1, int C1, int R2, int C2>
Matrix<S, R1, C2> operator*(const MBase<A, S, R1, C1>& a, const MBase<B, S, R2, C2>& b) {
    if (a.cols() != b.rows()) internal::fail("product dimension mismatch");
    Matrix<S, R1, C2> out;
    out.resize(a.rows(), b.cols());
    const Desc<S> x = a.desc(), y = b.desc(), o = out.desc();
    const Index n = x.c;
    if (n >= 16 && o.r * o.c >= 64) {
        // large operands: contiguous copies (rows of a, columns of b), same
        // sequential inner sums, so the result is identical to the loop below
        std::vector<S> ar(static_cast<size_t>(x.r * n)), bc(static_cast<size_t>(y.c * n));
        for (Index i = 0; i < x.r; ++i)
            for (Index k = 0; k < n; ++k) ar[i * n + k] = x.at(i, k);
        for (Index j = 0; j < y.c; ++j)
            for (Index k = 0; k < n; ++k) bc[j * n + k] = y.at(k, j);
        for (Index j = 0; j < o.c; ++j)
            for (Index i = 0; i < o.r; ++i) {
                const S* ap = &ar[i * n];
                const S* bp = &bc[j * n];
                S s = ap[0] * bp[0];
                for (Index k = 1; k < n; ++k) s += ap[k] * bp[k];
                o.at(i, j) = s;
            }
        return out;
    }
    for (Index j = 0; j < o.c; ++j)
        for (Index i = 0; i < o.r; ++i) {
            S s = n ? x.at(i, 0) * y.at(0, j) : S(0);
            for (Index k = 1; k < n; ++k) s += x.at(i, k) * y.at(k, j);
            o.at(i, j) = s;
        }
    return out;
}
template <class A, class S, int R, int C, int N>
Matrix<S, R, C> operator*(const MBase<A, S, R, C>& a, const DiagonalWrapper<S, N>& d) {
    if (a.cols() != d.rows()) internal::fail("diagonal product dimension mismatch");
    Matrix<S, R, C> out(a);
    for (Index j = 0; j < out.cols(); ++j)
        for (Index i = 0; i < out.rows(); ++i) out(i, j) = out(i, j) * d.diagonal()(j);
    return out;
}
template <class A, class S, int R, int C, int N>
Matrix<S, R, C> operator*(const DiagonalWrapper<S, N>& d, const MBase<A, S, R, C>& a) {
    if (a.rows() != d.cols()) internal::fail("diagonal product dimension mismatch");
    Matrix<S, R, C> out(a);
    for (Index j = 0; j < out.cols(); ++j)
        for (Index i = 0; i < out.rows(); ++i) out(i, j) = d.diagonal()(i) * out(i, j);
    return out;
}
template <class A, class B, class S, int R1, int C1, int R2, int C2>
bool operator==(const MBase<A, S, R1, C1>& a, const MBase<B, S, R2, C2>& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i)
            if (!(a.coeff(i, j) == b.coeff(i, j))) return false;
    return true;
}
template <class A, class B, class S, int R1, int C1, int R2, int C2>
bool operator!=(const MBase<A, S, R1, C1>& a, const MBase<B, S, R2, C2>& b) {
    return !(a == b);
}
template <class A, class S, int R, int C>
std::ostream& operator<<(std::ostream& os, const MBase<A, S, R, C>& m) {
    for (Index i = 0; i < m.rows(); ++i) {
        for (Index j = 0; j < m.cols(); ++j) os << (j ? " " : "") << m.coeff(i, j);
        if (i + 1 < m.rows()) os << "\n";
    }
    return os;
}

// ---------------------------------------------------------------------------
// decompositions
// ---------------------------------------------------------------------------
// LDLT<MatrixXd>: Eigen's ldlt_inplace<Lower>::unblocked — at step k the
// remaining diagonal entry of largest |.| is swapped in (symmetric pivoting,
// lower triangle only), then the column is formed left-looking; solve applies
// P, L^-1, D^+ (entries with |d| <= DBL_MIN give 0), L^-T, P^T.
template <class M>
class LDLT {
  public:
    using S = typename M::Scalar;
    LDLT() = default;
    template <class E, int R2, int C2>
    explicit LDLT(const MBase<E, S, R2, C2>& a) {
        compute(a);
    }
    template <class E, int R2, int C2>
    LDLT& compute(const MBase<E, S, R2, C2>& a) {
        if (a.rows() != a.cols()) internal::fail("LDLT of a non-square matrix");
        m_ = Matrix<S, Dynamic, Dynamic>(a);
        const Index n = m_.rows();
        tr_.assign(static_cast<size_t>(n), 0);
        std::vector<S> temp(static_cast<size_t>(n));
        bool ret = true, found_zero_pivot = false;
        for (Index k = 0; k < n; ++k) {
            Index big = k;
            S bigv = std::abs(m_(k, k));
            for (Index i = k + 1; i < n; ++i)
                if (std::abs(m_(i, i)) > bigv) {
                    bigv = std::abs(m_(i, i));
                    big = i;
                }
            tr_[k] = big;
            if (big != k) {
                const Index s = n - big - 1;
                for (Index j = 0; j < k; ++j) std::swap(m_(k, j), m_(big, j));
                for (Index i = 0; i < s; ++i) std::swap(m_(big + 1 + i, k), m_(big + 1 + i, big));
                std::swap(m_(k, k), m_(big, big));
                for (Index i = k + 1; i < big; ++i) {
                    const S tmp = m_(i, k);
                    m_(i, k) = m_(big, i);
                    m_(big, i) = tmp;
                }
            }
            const Index rs = n - k - 1;
            if (k > 0) {
                for (Index j = 0; j < k; ++j) temp[j] = m_(j, j) * m_(k, j);
                S dot = m_(k, 0) * temp[0];
                for (Index j = 1; j < k; ++j) dot += m_(k, j) * temp[j];
                m_(k, k) -= dot;
                for (Index i = 0; i < rs; ++i) {
                    S s = m_(k + 1 + i, 0) * temp[0];
                    for (Index j = 1; j < k; ++j) s += m_(k + 1 + i, j) * temp[j];
                    m_(k + 1 + i, k) -= s;
                }
            }
            const S akk = m_(k, k);
            const bool valid = std::abs(akk) > S(0);
            if (k == 0 && !valid) {  // the whole diagonal is zero
                for (Index j = 0; j < n; ++j) tr_[j] = j;
                info_ = Success;
                ok_ = true;
                return *this;
            }
            if (rs > 0 && valid) {
                for (Index i = 0; i < rs; ++i) m_(k + 1 + i, k) /= akk;
            } else if (rs > 0) {
                for (Index i = 0; i < rs; ++i) ret = ret && m_(k + 1 + i, k) == S(0);
            }
            if (found_zero_pivot && valid) ret = false;
            else if (!valid) found_zero_pivot = true;
        }
        info_ = ret ? Success : NumericalIssue;
        ok_ = true;
        return *this;
    }
    ComputationInfo info() const { return info_; }
    Matrix<S, Dynamic, 1> vectorD() const { return m_.diagonal(); }
    template <class E, int R2, int C2>
    Matrix<S, R2, C2> solve(const MBase<E, S, R2, C2>& b) const {
        if (!ok_) internal::fail("LDLT not initialised");
        const Index n = m_.rows();
        Matrix<S, R2, C2> x(b);
        for (Index c = 0; c < x.cols(); ++c) {
            for (Index k = 0; k < n; ++k) std::swap(x(k, c), x(tr_[k], c));
            for (Index k = 0; k < n; ++k)  // unit lower, column-oriented
                for (Index i = k + 1; i < n; ++i) x(i, c) -= x(k, c) * m_(i, k);
            const S tol = std::numeric_limits<S>::min();
            for (Index i = 0; i < n; ++i) x(i, c) = std::abs(m_(i, i)) > tol ? x(i, c) / m_(i, i) : S(0);
            for (Index i = n - 1; i >= 0; --i) {  // L^T, row-oriented
                S s = S(0);
                for (Index k = i + 1; k < n; ++k) s += m_(k, i) * x(k, c);
                x(i, c) -= s;
            }
            for (Index k = n - 1; k >= 0; --k) std::swap(x(k, c), x(tr_[k], c));
        }
        return x;
    }

  private:
    Matrix<S, Dynamic, Dynamic> m_;
    std::vector<Index> tr_;
    ComputationInfo info_ = InvalidInput;
    bool ok_ = false;
};

// FullPivLU: complete pivoting Gaussian elimination (rank-aware solve)
template <class M>
class FullPivLU {
  public:
    using S = typename M::Scalar;
    template <class E, int R2, int C2>
    explicit FullPivLU(const MBase<E, S, R2, C2>& a) : lu_(a) {
        const Index n = lu_.rows(), m = lu_.cols(), k_max = std::min(n, m);
        rp_.resize(static_cast<size_t>(n));
        cp_.resize(static_cast<size_t>(m));
        for (Index i = 0; i < n; ++i) rp_[i] = i;
        for (Index j = 0; j < m; ++j) cp_[j] = j;
        S maxpivot = 0;
        rank_ = 0;
        for (Index k = 0; k < k_max; ++k) {
            Index bi = k, bj = k;
            S best = -1;
            for (Index j = k; j < m; ++j)
                for (Index i = k; i < n; ++i)
                    if (std::abs(lu_(i, j)) > best) best = std::abs(lu_(i, j)), bi = i, bj = j;
            if (best == S(0)) break;
            maxpivot = std::max(maxpivot, best);
            if (bi != k) {
                for (Index j = 0; j < m; ++j) std::swap(lu_(k, j), lu_(bi, j));
                std::swap(rp_[k], rp_[bi]);
            }
            if (bj != k) {
                for (Index i = 0; i < n; ++i) std::swap(lu_(i, k), lu_(i, bj));
                std::swap(cp_[k], cp_[bj]);
            }
            for (Index i = k + 1; i < n; ++i) {
                lu_(i, k) /= lu_(k, k);
                for (Index j = k + 1; j < m; ++j) lu_(i, j) -= lu_(i, k) * lu_(k, j);
            }
            ++rank_;
        }
        const S thr = std::numeric_limits<S>::epsilon() * S(k_max) * maxpivot;
        Index r = 0;
        for (Index k = 0; k < rank_; ++k)
            if (std::abs(lu_(k, k)) > thr) ++r;
        rank_ = r;
    }
    Index rank() const { return rank_; }
    bool isInvertible() const { return rank_ == lu_.rows() && lu_.rows() == lu_.cols(); }
    template <class E, int R2, int C2>
    Matrix<S, Dynamic, C2> solve(const MBase<E, S, R2, C2>& b) const {
        const Index n = lu_.rows(), m = lu_.cols();
        Matrix<S, Dynamic, C2> x;
        x.resize(m, b.cols());
        for (Index c = 0; c < b.cols(); ++c) {
            std::vector<S> y(static_cast<size_t>(n));
            for (Index i = 0; i < n; ++i) y[i] = b.coeff(rp_[i], c);
            for (Index i = 0; i < rank_; ++i)
                for (Index k = 0; k < i; ++k) y[i] -= lu_(i, k) * y[k];
            std::vector<S> z(static_cast<size_t>(m), S(0));
            for (Index i = rank_ - 1; i >= 0; --i) {
                S s = y[i];
                for (Index k = i + 1; k < rank_; ++k) s -= lu_(i, k) * z[k];
                z[i] = s / lu_(i, i);
            }
            for (Index j = 0; j < m; ++j) x(cp_[j], c) = z[j];
        }
        return x;
    }

  private:
    Matrix<S, Dynamic, Dynamic> lu_;
    std::vector<Index> rp_, cp_;
    Index rank_ = 0;
};

// ColPivHouseholderQR: Householder QR with column pivoting by remaining norm
template <class M>
class ColPivHouseholderQR {
  public:
    using S = typename M::Scalar;
    template <class E, int R2, int C2>
    explicit ColPivHouseholderQR(const MBase<E, S, R2, C2>& a) : qr_(a) {
        const Index n = qr_.rows(), m = qr_.cols(), k_max = std::min(n, m);
        perm_.resize(static_cast<size_t>(m));
        for (Index j = 0; j < m; ++j) perm_[j] = j;
        tau_.assign(static_cast<size_t>(k_max), S(0));
        S maxpivot = 0;
        for (Index k = 0; k < k_max; ++k) {
            Index bj = k;
            S best = -1;
            for (Index j = k; j < m; ++j) {
                S s = 0;
                for (Index i = k; i < n; ++i) s += qr_(i, j) * qr_(i, j);
                if (s > best) best = s, bj = j;
            }
            if (bj != k) {
                for (Index i = 0; i < n; ++i) std::swap(qr_(i, k), qr_(i, bj));
                std::swap(perm_[k], perm_[bj]);
            }
            S norm = 0;
            for (Index i = k; i < n; ++i) norm += qr_(i, k) * qr_(i, k);
            norm = std::sqrt(norm);
            if (norm == S(0)) continue;
            const S alpha = qr_(k, k) > 0 ? -norm : norm;
            const S v0 = qr_(k, k) - alpha;
            for (Index i = k + 1; i < n; ++i) qr_(i, k) /= v0;  // v = [1, qr(k+1:, k)]
            tau_[k] = -v0 / alpha;  // LAPACK's (beta - x0) / beta with beta = alpha
            qr_(k, k) = alpha;
            maxpivot = std::max(maxpivot, std::abs(alpha));
            for (Index j = k + 1; j < m; ++j) {
                S s = qr_(k, j);
                for (Index i = k + 1; i < n; ++i) s += qr_(i, k) * qr_(i, j);
                s *= tau_[k];
                qr_(k, j) -= s;
                for (Index i = k + 1; i < n; ++i) qr_(i, j) -= s * qr_(i, k);
            }
        }
        const S thr = std::numeric_limits<S>::epsilon() * S(k_max) * maxpivot;
        rank_ = 0;
        for (Index k = 0; k < k_max; ++k)
            if (std::abs(qr_(k, k)) > thr) ++rank_;
    }
    template <class E, int R2, int C2>
    Matrix<S, Dynamic, C2> solve(const MBase<E, S, R2, C2>& b) const {
        const Index n = qr_.rows(), m = qr_.cols();
        Matrix<S, Dynamic, C2> x;
        x.resize(m, b.cols());
        for (Index c = 0; c < b.cols(); ++c) {
            std::vector<S> y(static_cast<size_t>(n));
            for (Index i = 0; i < n; ++i) y[i] = b.coeff(i, c);
            for (Index k = 0; k < static_cast<Index>(tau_.size()); ++k) {  // y = Q^T b
                S s = y[k];
                for (Index i = k + 1; i < n; ++i) s += qr_(i, k) * y[i];
                s *= tau_[k];
                y[k] -= s;
                for (Index i = k + 1; i < n; ++i) y[i] -= s * qr_(i, k);
            }
            std::vector<S> z(static_cast<size_t>(m), S(0));
            for (Index i = rank_ - 1; i >= 0; --i) {
                S s = y[i];
                for (Index k = i + 1; k < rank_; ++k) s -= qr_(i, k) * z[k];
                z[i] = s / qr_(i, i);
            }
            for (Index j = 0; j < m; ++j) x(perm_[j], c) = z[j];
        }
        return x;
    }

  private:
    Matrix<S, Dynamic, Dynamic> qr_;
    std::vector<Index> perm_;
    std::vector<S> tau_;
    Index rank_ = 0;
};

template <class D, class S, int R, int C>
LDLT<Matrix<S, R, C>> MBase<D, S, R, C>::ldlt() const {
    return LDLT<Matrix<S, R, C>>(*this);
}
template <class D, class S, int R, int C>
FullPivLU<Matrix<S, R, C>> MBase<D, S, R, C>::fullPivLu() const {
    return FullPivLU<Matrix<S, R, C>>(*this);
}
template <class D, class S, int R, int C>
ColPivHouseholderQR<Matrix<S, R, C>> MBase<D, S, R, C>::colPivHouseholderQr() const {
    return ColPivHouseholderQR<Matrix<S, R, C>>(*this);
}
template <class D, class S, int R, int C>
typename MBase<D, S, R, C>::PlainObject MBase<D, S, R, C>::inverse() const {
    if (rows() != cols()) internal::fail("inverse of a non-square matrix");
    const FullPivLU<Matrix<S, Dynamic, Dynamic>> lu(*this);
    return PlainObject(lu.solve(Matrix<S, Dynamic, Dynamic>::Identity(rows(), cols())));
}
template <class D, class S, int R, int C>
S MBase<D, S, R, C>::determinant() const {
    if (rows() != cols()) internal::fail("determinant of a non-square matrix");
    Matrix<S, Dynamic, Dynamic> a(*this);
    const Index n = a.rows();
    S det = 1;
    for (Index k = 0; k < n; ++k) {
        Index p = k;
        for (Index i = k + 1; i < n; ++i)
            if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
        if (a(p, k) == S(0)) return S(0);
        if (p != k) {
            for (Index j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
            det = -det;
        }
        det *= a(k, k);
        for (Index i = k + 1; i < n; ++i) {
            const S f = a(i, k) / a(k, k);
            for (Index j = k + 1; j < n; ++j) a(i, j) -= f * a(k, j);
        }
    }
    return det;
}

// JacobiSVD (3x3 use in trajectory alignment): one-sided Jacobi, singular
// values sorted decreasingly, U completed for rank-deficient inputs
template <class M>
class JacobiSVD {
  public:
    using S = typename M::Scalar;
    template <class E, int R2, int C2>
    JacobiSVD(const MBase<E, S, R2, C2>& a, unsigned = 0) {
        const Index n = a.rows(), m = a.cols();
        Matrix<S, Dynamic, Dynamic> A(a);
        Matrix<S, Dynamic, Dynamic> V = Matrix<S, Dynamic, Dynamic>::Identity(m, m);
        for (int sweep = 0; sweep < 60; ++sweep) {
            bool rotated = false;
            for (Index p = 0; p < m; ++p)
                for (Index q = p + 1; q < m; ++q) {
                    S al = 0, be = 0, ga = 0;
                    for (Index i = 0; i < n; ++i) {
                        al += A(i, p) * A(i, p);
                        be += A(i, q) * A(i, q);
                        ga += A(i, p) * A(i, q);
                    }
                    if (std::abs(ga) <= std::numeric_limits<S>::epsilon() * std::sqrt(al * be) || ga == S(0)) continue;
                    rotated = true;
                    const S zeta = (be - al) / (2 * ga);
                    const S t = (zeta >= 0 ? S(1) : S(-1)) / (std::abs(zeta) + std::sqrt(S(1) + zeta * zeta));
                    const S c = S(1) / std::sqrt(S(1) + t * t), s = c * t;
                    for (Index i = 0; i < n; ++i) {
                        const S x = A(i, p), y = A(i, q);
                        A(i, p) = c * x - s * y;
                        A(i, q) = s * x + c * y;
                    }
                    for (Index i = 0; i < m; ++i) {
                        const S x = V(i, p), y = V(i, q);
                        V(i, p) = c * x - s * y;
                        V(i, q) = s * x + c * y;
                    }
                }
            if (!rotated) break;
        }
        std::vector<Index> order(static_cast<size_t>(m));
        std::vector<S> sv(static_cast<size_t>(m));
        for (Index j = 0; j < m; ++j) {
            order[j] = j;
            sv[j] = A.col(j).norm();
        }
        std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return sv[x] > sv[y]; });
        s_.resize(m);
        u_.resize(n, n);
        v_.resize(m, m);
        u_.setZero();
        for (Index k = 0; k < m; ++k) {
            const Index j = order[k];
            s_(k) = sv[j];
            v_.col(k) = V.col(j);
            if (k < n && sv[j] > std::numeric_limits<S>::min()) u_.col(k) = A.col(j) / sv[j];
        }
        for (Index k = 0; k < n; ++k) {  // complete U by Gram-Schmidt on unit vectors
            if (u_.col(k).squaredNorm() > S(0.5)) continue;
            for (Index e = 0; e < n; ++e) {
                Matrix<S, Dynamic, 1> cand = Matrix<S, Dynamic, 1>::Zero(n);
                cand(e) = 1;
                for (Index o = 0; o < n; ++o)
                    if (o != k && u_.col(o).squaredNorm() > S(0.5)) cand -= u_.col(o).dot(cand) * u_.col(o);
                if (cand.norm() > S(1e-6)) {
                    u_.col(k) = cand.normalized();
                    break;
                }
            }
        }
    }
    const Matrix<S, Dynamic, Dynamic>& matrixU() const { return u_; }
    const Matrix<S, Dynamic, Dynamic>& matrixV() const { return v_; }
    const Matrix<S, Dynamic, 1>& singularValues() const { return s_; }

  private:
    Matrix<S, Dynamic, Dynamic> u_, v_;
    Matrix<S, Dynamic, 1> s_;
};

// ---------------------------------------------------------------------------
// typedefs
// ---------------------------------------------------------------------------
#define PVO_SHIM_TYPEDEFS(S, suffix)                        \
    using Matrix2##suffix = Matrix<S, 2, 2>;                \
    using Matrix3##suffix = Matrix<S, 3, 3>;                \
    using Matrix4##suffix = Matrix<S, 4, 4>;                \
    using MatrixX##suffix = Matrix<S, Dynamic, Dynamic>;    \
    using Vector2##suffix = Matrix<S, 2, 1>;                \
    using Vector3##suffix = Matrix<S, 3, 1>;                \
    using Vector4##suffix = Matrix<S, 4, 1>;                \
    using VectorX##suffix = Matrix<S, Dynamic, 1>;          \
    using RowVector2##suffix = Matrix<S, 1, 2>;             \
    using RowVector3##suffix = Matrix<S, 1, 3>;             \
    using RowVectorX##suffix = Matrix<S, 1, Dynamic>;
PVO_SHIM_TYPEDEFS(double, d)
PVO_SHIM_TYPEDEFS(float, f)
PVO_SHIM_TYPEDEFS(int, i)
#undef PVO_SHIM_TYPEDEFS
template <class S, int N>
using Vector = Matrix<S, N, 1>;

// ---------------------------------------------------------------------------
// Quaternion (Geometry/Quaternion.h): coeffs stored (x, y, z, w)
// ---------------------------------------------------------------------------
template <class S>
class Quaternion {
  public:
    using Scalar = S;
    using Vector3 = Matrix<S, 3, 1>;
    using Coefficients = Matrix<S, 4, 1>;
    Quaternion() = default;
    Quaternion(S w, S x, S y, S z) : c_(x, y, z, w) {}
    explicit Quaternion(const Coefficients& c) : c_(c) {}
    template <class E, int R2, int C2>
    explicit Quaternion(const MBase<E, S, R2, C2>& m) {
        if (m.rows() == 3 && m.cols() == 3) from_rotation(Matrix<S, 3, 3>(m));
        else c_ = Coefficients(m);
    }
    static Quaternion Identity() { return Quaternion(S(1), S(0), S(0), S(0)); }

    S& w() { return c_(3); }
    S& x() { return c_(0); }
    S& y() { return c_(1); }
    S& z() { return c_(2); }
    S w() const { return c_(3); }
    S x() const { return c_(0); }
    S y() const { return c_(1); }
    S z() const { return c_(2); }
    Coefficients& coeffs() { return c_; }
    const Coefficients& coeffs() const { return c_; }
    View<S, 3, 1> vec() const { return c_.template head<3>(); }

    S squaredNorm() const { return c_.squaredNorm(); }
    S norm() const { return c_.norm(); }
    void normalize() { c_.normalize(); }
    Quaternion normalized() const { return Quaternion(c_.normalized()); }
    S dot(const Quaternion& o) const { return c_.dot(o.c_); }
    Quaternion conjugate() const { return Quaternion(c_(3), -c_(0), -c_(1), -c_(2)); }
    Quaternion inverse() const {
        const S n2 = squaredNorm();
        if (n2 > S(0)) {
            Quaternion q = conjugate();
            q.c_ /= n2;
            return q;
        }
        return Quaternion(Coefficients::Zero());
    }
    S angularDistance(const Quaternion& o) const {
        const Quaternion d = (*this) * o.conjugate();
        return S(2) * std::atan2(d.vec().norm(), std::abs(d.w()));
    }
    // quat_product (Quaternion.h, generic path)
    Quaternion operator*(const Quaternion& b) const {
        const Quaternion& a = *this;
        return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                          a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                          a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                          a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
    }
    Quaternion& operator*=(const Quaternion& b) { return *this = (*this) * b; }
    // _transformVector: uv = 2 vec x v; v + w uv + vec x uv
    template <class E, int R2, int C2>
    Vector3 operator*(const MBase<E, S, R2, C2>& v_in) const {
        const Vector3 v(v_in);
        const Vector3 qv(x(), y(), z());
        Vector3 uv = qv.cross(v);
        uv += uv;
        return v + w() * uv + qv.cross(uv);
    }
    Matrix<S, 3, 3> toRotationMatrix() const {
        Matrix<S, 3, 3> res;
        const S tx = S(2) * x(), ty = S(2) * y(), tz = S(2) * z();
        const S twx = tx * w(), twy = ty * w(), twz = tz * w();
        const S txx = tx * x(), txy = ty * x(), txz = tz * x();
        const S tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
        res(0, 0) = S(1) - (tyy + tzz);
        res(0, 1) = txy - twz;
        res(0, 2) = txz + twy;
        res(1, 0) = txy + twz;
        res(1, 1) = S(1) - (txx + tzz);
        res(1, 2) = tyz - twx;
        res(2, 0) = txz - twy;
        res(2, 1) = tyz + twx;
        res(2, 2) = S(1) - (txx + tyy);
        return res;
    }
    Matrix<S, 3, 3> matrix() const { return toRotationMatrix(); }
    template <class E, int R2, int C2>
    Quaternion& operator=(const MBase<E, S, R2, C2>& m) {
        from_rotation(Matrix<S, 3, 3>(m));
        return *this;
    }

  private:
    // quaternionbase_assign_impl<Other, 3, 3>
    void from_rotation(const Matrix<S, 3, 3>& m) {
        const S t = m.trace();
        if (t > S(0)) {
            S r = std::sqrt(t + S(1));
            w() = S(0.5) * r;
            r = S(0.5) / r;
            x() = (m(2, 1) - m(1, 2)) * r;
            y() = (m(0, 2) - m(2, 0)) * r;
            z() = (m(1, 0) - m(0, 1)) * r;
        } else {
            Index i = 0;
            if (m(1, 1) > m(0, 0)) i = 1;
            if (m(2, 2) > m(i, i)) i = 2;
            const Index j = (i + 1) % 3, k = (j + 1) % 3;
            S r = std::sqrt(m(i, i) - m(j, j) - m(k, k) + S(1));
            c_(i) = S(0.5) * r;
            r = S(0.5) / r;
            w() = (m(k, j) - m(j, k)) * r;
            c_(j) = (m(j, i) + m(i, j)) * r;
            c_(k) = (m(k, i) + m(i, k)) * r;
        }
    }
    Coefficients c_ = Coefficients(S(0), S(0), S(0), S(1));
};
using Quaterniond = Quaternion<double>;
using Quaternionf = Quaternion<float>;

}  // namespace Eigen
