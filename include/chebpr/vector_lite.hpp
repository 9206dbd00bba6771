// Minimal stand-in for Eigen::VectorXd, used by the drop-in headers when Eigen is not on
// the include path (it is absent from this image).  Provides exactly the subset the
// reference API and its tests use: Ones/Constant/Zero, (n) construction, size/resize,
// data, [] and (), swap, comma initialisation and maxCoeff(&index).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <type_traits>
#include <vector>

namespace chebpr {

class VectorLite {
public:
    using Index = std::ptrdiff_t;
    VectorLite() = default;
    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    explicit VectorLite(I n) : v_(static_cast<size_t>(n), 0.0) {}

    static VectorLite Constant(Index n, double x) {
        VectorLite r(n);
        std::fill(r.v_.begin(), r.v_.end(), x);
        return r;
    }
    static VectorLite Ones(Index n) { return Constant(n, 1.0); }
    static VectorLite Zero(Index n) { return Constant(n, 0.0); }

    Index size() const { return static_cast<Index>(v_.size()); }
    void resize(Index n) { v_.resize(static_cast<size_t>(n)); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
    double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
    double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
    void swap(VectorLite& o) { v_.swap(o.v_); }

    class Filler {
    public:
        Filler(VectorLite& v, double first) : v_(v) { v_[pos_++] = first; }
        Filler& operator,(double x) {
            v_[pos_++] = x;
            return *this;
        }

    private:
        VectorLite& v_;
        Index pos_ = 0;
    };
    Filler operator<<(double x) { return Filler(*this, x); }

    template <class I>
    double maxCoeff(I* where) const {
        const auto it = std::max_element(v_.begin(), v_.end());
        *where = static_cast<I>(it - v_.begin());
        return *it;
    }

private:
    std::vector<double> v_;
};

}  // namespace chebpr
