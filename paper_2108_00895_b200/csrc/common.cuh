// Shared helpers for the sskm_b200 CUDA engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "sskm_b200 is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace sskm_b200 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw CudaError(std::string("CUDA error in ") + what + " (" + file + ":" +
                        std::to_string(line) + "): " + cudaGetErrorString(e));
    }
}
#define CK(x) ::sskm_b200::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::sskm_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

constexpr uint32_t kNone = 0xFFFFFFFFu;  // "no cluster" marker for the sums' owner map
constexpr int kWarp = 32;

// Lexicographic (sim desc, id asc) — the reference tie rule
// `s > best || (s == best && j < arg)` (engine.cpp:259) as a total order, so
// any reduction order yields the reference's sequential result.
__device__ __forceinline__ bool better(double s, uint32_t j, double best, uint32_t arg) {
    return s > best || (s == best && j < arg);
}

__device__ __forceinline__ void warp_argmax(double& best, uint32_t& arg) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        uint32_t oa = __shfl_xor_sync(0xFFFFFFFFu, arg, off);
        if (better(ob, oa, best, arg)) {
            best = ob;
            arg = oa;
        }
    }
}

// Monotone map of a double onto uint64 (for atomicMin on fp64 keys).
__device__ __forceinline__ unsigned long long orderable(double x) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

}  // namespace sskm_b200
