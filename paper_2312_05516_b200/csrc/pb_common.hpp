// Shared host-side helpers: status/error plumbing and launch accounting.
#pragma once

#include "pensieve_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
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
// While alive, this thread's count_launch calls add to `n` instead of the process counter
// (kernels captured into a graph are counted per graph launch).
struct LaunchCapture {
    uint64_t n = 0;
    LaunchCapture();
    ~LaunchCapture();
    LaunchCapture(const LaunchCapture&) = delete;
    LaunchCapture& operator=(const LaunchCapture&) = delete;

  private:
    uint64_t* prev_;
};

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

// ---- per-device state (one host thread per GPU is the multi-GPU control plane)
// Kernel attributes such as the dynamic shared-memory opt-in are per device, so they are set
// once per (kernel, device) under std::call_once; SM counts are cached per device.
constexpr int kMaxDevices = 64;

inline int current_device() {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) fail(PB_ERR_UNSUPPORTED, "device ordinal out of range");
    return dev;
}

// SM count of the current device (148 on B200).  With no usable device (host-only plan
// building in the CPU container) the B200 count is returned.
int device_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).  `flags` is the
// per-kernel once-table (a function-local static in the launcher).
template <class K>
inline void set_smem_once(std::once_flag (&flags)[kMaxDevices], K kernel, size_t bytes, const char* what) {
    const int dev = current_device();
    std::call_once(flags[dev], [&] {
        cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
                   what);
    });
}

} // namespace pb
