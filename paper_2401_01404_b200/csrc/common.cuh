// common.cuh — shared device helpers for libnetrec_b200 (sm_100a).
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace nrg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

#define NRG_CUDA(x)                                                                     \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            ::nrg::fail(100, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " +  \
                                 __FILE__ + ":" + std::to_string(__LINE__));            \
    } while (0)
// every kernel launch site is followed by NRG_LAUNCH_CHECK(n_launches)
inline std::atomic<uint64_t> g_launches{0};
#define NRG_LAUNCH_CHECK_N(k)                \
    do {                                     \
        ::nrg::g_launches += (k);            \
        NRG_CUDA(cudaGetLastError());        \
    } while (0)
#define NRG_LAUNCH_CHECK() NRG_LAUNCH_CHECK_N(1)

// ---------------------------------------------------------------- keys
// pair_key (inc/common.hpp:33-37): (min << 32) | max
__host__ __device__ __forceinline__ uint64_t pair_key(int32_t a, int32_t b) {
    if (a > b) {
        int32_t t = a;
        a = b;
        b = t;
    }
    return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}

// order-preserving map double -> uint64 (total order for finite doubles, -0 < +0)
__host__ __device__ __forceinline__ uint64_t dkey(double d) {
    uint64_t u;
#ifdef __CUDA_ARCH__
    u = (uint64_t)__double_as_longlong(d);
#else
    __builtin_memcpy(&u, &d, 8);
#endif
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__host__ __device__ __forceinline__ double dkey_inv(uint64_t k) {
    uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
    double d;
#ifdef __CUDA_ARCH__
    d = __longlong_as_double((long long)u);
#else
    __builtin_memcpy(&d, &u, 8);
#endif
    return d;
}

// ---------------------------------------------------------------- RNG
// SplitMix64 finalizer and SplitRng (inc/random.hpp:11-65)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }

struct SplitRng {
    uint64_t key, ctr;
    __host__ __device__ explicit SplitRng(uint64_t seed = 0) : key(mix64(seed)), ctr(0) {}
    __host__ __device__ SplitRng split(uint64_t stream) const {
        SplitRng r;
        r.key = mix64(key, stream);
        r.ctr = 0;
        return r;
    }
    __host__ __device__ uint64_t next() { return mix64(key + 0x9e3779b97f4a7c15ULL * ++ctr); }
    __host__ __device__ double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    // Lemire 128-bit multiply (inc/random.hpp:48-52)
    __host__ __device__ uint64_t below(uint64_t n) {
#ifdef __CUDA_ARCH__
        return __umul64hi(next(), n);
#else
        return (uint64_t)(((unsigned __int128)next() * n) >> 64);
#endif
    }
};

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr uint64_t kEmptyKey = 0xffffffffffffffffULL;
constexpr uint64_t kTombKey = 0xfffffffffffffffeULL;

// home slot of a pair key in the open-addressing tables (couplings W, distance cache):
// Fibonacci hashing, bits 32..63 of key * 2^64/phi (one 64-bit multiply; both node
// ids reach those bits), masked to a power-of-two capacity <= 2^32
__host__ __device__ __forceinline__ uint64_t slot_of(uint64_t key, uint64_t mask) {
    return ((key * 0x9e3779b97f4a7c15ULL) >> 32) & mask;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// A/B and debug switches read once per call site (getenv scans the environment; several
// sit on per-sweep paths).  Switches the tests toggle in-process keep plain getenv.
#define NRG_ENV_ON(name) ([] { static const bool v_ = getenv(name) != nullptr; return v_; }())

}  // namespace nrg
