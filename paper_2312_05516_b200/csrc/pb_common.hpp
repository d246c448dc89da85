// Shared host-side helpers: status/error plumbing and launch accounting.
#pragma once

#include "pensieve_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace pb {

// Thrown internally, converted to a pb_status at the C-ABI boundary (no exception ever
// crosses extern "C").  Mirrors the reference's exception hierarchy
// (include/kvsim/errors.hpp) one class per status code.
struct Failure : std::runtime_error {
    pb_status code;
    Failure(pb_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(pb_status c, const std::string& msg) { throw Failure(c, msg); }

inline void require(bool ok, const char* what) {
    if (!ok) fail(PB_ERR_DIMENSION_MISMATCH, what);
}

void set_last_error(const std::string& msg);
void count_launch(uint64_t n = 1);

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(PB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs f, mapping Failure / CUDA / allocation errors onto status codes.
template <class F> pb_status guarded(F&& f) {
    try {
        f();
        return PB_OK;
    } catch (const Failure& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return PB_ERR_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PB_ERR_ERROR;
    }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

} // namespace pb
