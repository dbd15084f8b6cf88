// Exception hierarchy of the drop-in API: the same types, in the same
// namespace, as the reference (proj/include/bcad/errors.hpp:8-66), plus the
// mapping from C-ABI status codes (include/bcad_cu.h) back to them.
#pragma once

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "bcad_cu.h"

namespace bcad {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TagMismatch : Error { using Error::Error; };
struct DivisionByZero : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct NonDifferentiablePoint : Error { using Error::Error; };
struct ShapeMismatch : Error { using Error::Error; };
struct ArityMismatch : Error { using Error::Error; };
struct SeedShapeMismatch : Error { using Error::Error; };
struct UnknownPrimitive : Error { using Error::Error; };
struct NonFiniteValue : Error { using Error::Error; };
struct SizeGuardExceeded : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct EquivalenceFailure : Error { using Error::Error; };
// Device-side failures have no reference counterpart.
struct CudaError : Error { using Error::Error; };
struct NcclError : Error { using Error::Error; };

[[noreturn]] inline void throw_status(int code, const std::string& msg) {
    switch (code) {
        case BCAD_CU_ERR_TAG_MISMATCH: throw TagMismatch(msg);
        case BCAD_CU_ERR_DIVISION_BY_ZERO: throw DivisionByZero(msg);
        case BCAD_CU_ERR_DOMAIN: throw DomainError(msg);
        case BCAD_CU_ERR_NON_DIFFERENTIABLE: throw NonDifferentiablePoint(msg);
        case BCAD_CU_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case BCAD_CU_ERR_ARITY_MISMATCH: throw ArityMismatch(msg);
        case BCAD_CU_ERR_SEED_SHAPE_MISMATCH: throw SeedShapeMismatch(msg);
        case BCAD_CU_ERR_UNKNOWN_PRIMITIVE: throw UnknownPrimitive(msg);
        case BCAD_CU_ERR_NON_FINITE: throw NonFiniteValue(msg);
        case BCAD_CU_ERR_SIZE_GUARD: throw SizeGuardExceeded(msg);
        case BCAD_CU_ERR_CONFIG: throw ConfigError(msg);
        case BCAD_CU_ERR_IO: throw IoError(msg);
        case BCAD_CU_ERR_EQUIVALENCE: throw EquivalenceFailure(msg);
        case BCAD_CU_ERR_CUDA: throw CudaError(msg);
        case BCAD_CU_ERR_NCCL: throw NcclError(msg);
        default: throw Error(msg);
    }
}

// Generation of device memory as the host API sees it. Any C-ABI call made
// through check() may have written device memory (or enqueued a write), so it
// advances the generation; a Tensor's cached host view of its elements
// (tensor.hpp, element reads) is valid only within the generation it was
// taken in.
inline std::atomic<std::uint64_t>& device_generation() {
    static std::atomic<std::uint64_t> g{1};
    return g;
}
inline void advance_device_generation() { device_generation().fetch_add(1, std::memory_order_relaxed); }

// Throws the bcad exception matching a non-OK C-ABI status.
inline void check(int status) {
    advance_device_generation();
    if (status != BCAD_CU_OK) throw_status(status, bcad_cu_last_error());
}

// The same for calls that only read device memory into the host (a cached
// element view must not invalidate itself).
inline void check_read(int status) {
    if (status != BCAD_CU_OK) throw_status(status, bcad_cu_last_error());
}

}  // namespace bcad
