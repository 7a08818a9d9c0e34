#pragma once
// Exception hierarchy of the drop-in API — same class names, members and
// accessors as the reference (errors.hpp:10-113).  Device-side failures are
// reported through the C-ABI (pswarm_error) and rethrown as these types by
// throw_from_status(); CUDA failures raise DeviceError (no reference analogue).

#include <cstdint>
#include <stdexcept>
#include <string>

#include "pswarm_gpu.h"

namespace pswarm {

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class InvalidSpanError : public Error { public: using Error::Error; };
class InvalidSizeError : public Error { public: using Error::Error; };
class ShapeError : public Error { public: using Error::Error; };
class AlignmentError : public Error { public: using Error::Error; };

class DivergenceError : public Error {
public:
    DivergenceError(const std::string& what, std::int64_t node, std::int64_t column)
        : Error(what), node_(node), column_(column) {}
    std::int64_t node() const noexcept { return node_; }
    std::int64_t column() const noexcept { return column_; }

private:
    std::int64_t node_;
    std::int64_t column_;
};

class SingularityError : public Error {
public:
    explicit SingularityError(const std::string& what, std::string body = {}) : Error(what), body_(std::move(body)) {}
    const std::string& body() const noexcept { return body_; }

private:
    std::string body_;
};

class CoverageError : public Error {
public:
    CoverageError(const std::string& what, double epoch) : Error(what), epoch_(epoch) {}
    double epoch() const noexcept { return epoch_; }

private:
    double epoch_;
};

class NonEllipticError : public Error { public: using Error::Error; };
class SolverError : public Error { public: using Error::Error; };
class InvalidPlanError : public Error { public: using Error::Error; };
class EmptyReductionError : public Error { public: using Error::Error; };
class OracleError : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
class TimeoutError : public Error { public: using Error::Error; };

/// CUDA / device failure (no CPU fallback exists; the call cannot be completed).
class DeviceError : public Error { public: using Error::Error; };

/// Rethrows a C-ABI failure as the matching reference exception type.
/// PSWARM_ERR_INCOMPLETE is handled by the propagator (it carries a partial result).
[[noreturn]] inline void throw_from_status(const pswarm_error& e) {
    const std::string m = e.message;
    switch (e.status) {
    case PSWARM_ERR_INVALID_SPAN: throw InvalidSpanError(m);
    case PSWARM_ERR_INVALID_SIZE: throw InvalidSizeError(m);
    case PSWARM_ERR_SHAPE: throw ShapeError(m);
    case PSWARM_ERR_ALIGNMENT: throw AlignmentError(m);
    case PSWARM_ERR_DIVERGENCE: throw DivergenceError(m, e.node, e.column);
    case PSWARM_ERR_SINGULARITY: throw SingularityError(m, e.body_name);
    case PSWARM_ERR_COVERAGE: throw CoverageError(m, e.value);
    case PSWARM_ERR_NON_ELLIPTIC: throw NonEllipticError(m);
    case PSWARM_ERR_SOLVER: throw SolverError(m);
    case PSWARM_ERR_INVALID_PLAN: throw InvalidPlanError(m);
    case PSWARM_ERR_EMPTY_REDUCTION: throw EmptyReductionError(m);
    case PSWARM_ERR_TIMEOUT: throw TimeoutError(m);
    case PSWARM_ERR_ORACLE: throw OracleError(m);
    case PSWARM_ERR_CUDA:
    case PSWARM_ERR_OOM:
    case PSWARM_ERR_NO_DEVICE: throw DeviceError(m);
    default: throw Error(m);
    }
}

}  // namespace pswarm
