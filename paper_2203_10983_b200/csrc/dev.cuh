// dev.cuh -- device helpers shared by the kernels (16-byte vector rows of fp32 or bf16).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <utility>

namespace bns {

// Programmatic dependent launch (PDL).  Every kernel of the library starts with pdl_grid_sync(): wait until the
// previous grid in the stream has completed and its writes are visible (griddepcontrol.wait -- a no-op when the
// kernel was launched without the PDL attribute), then let the next grid's CTAs be scheduled (launch_dependents).
// Launched by pdl_launch, a kernel's CTAs therefore become resident while the previous kernel drains and start the
// moment it completes: the launch latency and the CTA ramp of each of the ~50 kernels of an epoch overlap the tail
// of the one before.  Because each grid waits before it touches memory and triggers only after that wait, a grid's
// completion still implies the completion of everything enqueued before it (the usual stream order).
__device__ __forceinline__ void pdl_grid_sync() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// BNS_PDL=0 launches every kernel with plain stream serialisation (A/B); pdl_take_hold (common.h): this launch
// follows a non-kernel stream operation
bool pdl_enabled();
bool pdl_take_hold();

template <typename... KArgs, typename... Args>
inline void pdl_launch(cudaStream_t s, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (!pdl_take_hold() && pdl_enabled()) ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);   // errors surface in BNS_CHECK_LAUNCH
}

// A 16-byte vector of the storage type: 4 x fp32 or 8 x bf16.
template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int N = 4;
    using raw = float4;
    __device__ __forceinline__ static void add_scaled(float* acc, const raw& v, float s) {
        acc[0] = fmaf(s, v.x, acc[0]); acc[1] = fmaf(s, v.y, acc[1]);
        acc[2] = fmaf(s, v.z, acc[2]); acc[3] = fmaf(s, v.w, acc[3]);
    }
    __device__ __forceinline__ static void to_float(const raw& v, float* f) { f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w; }
    __device__ __forceinline__ static raw from_float(const float* f) { return make_float4(f[0], f[1], f[2], f[3]); }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    using raw = uint4;
    __device__ __forceinline__ static void add_scaled(float* acc, const raw& v, float s) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float lo = __uint_as_float(w[k] << 16), hi = __uint_as_float(w[k] & 0xffff0000u);
            acc[2 * k] = fmaf(s, lo, acc[2 * k]);
            acc[2 * k + 1] = fmaf(s, hi, acc[2 * k + 1]);
        }
    }
    __device__ __forceinline__ static void to_float(const raw& v, float* f) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) { f[2 * k] = __uint_as_float(w[k] << 16); f[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u); }
    }
    __device__ __forceinline__ static raw from_float(const float* f) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
            w[k] = *reinterpret_cast<uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};

// Packed fp32x2 accumulate (sm_100 FFMA2 / FADD2): acc[0..1] += s * (x, y)  /  acc[0..1] += (x, y)
__device__ __forceinline__ void ffma2(float* acc, float x, float y, float s) {
    uint64_t c, a, b;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(acc[0]), "f"(acc[1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(x), "f"(y));
    asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[0]), "=f"(acc[1]) : "l"(c));
}
__device__ __forceinline__ void fadd2(float* acc, float x, float y) {
    uint64_t c, a;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(acc[0]), "f"(acc[1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(x), "f"(y));
    asm("add.rn.f32x2 %0, %1, %0;" : "+l"(c) : "l"(a));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[0]), "=f"(acc[1]) : "l"(c));
}
// Packed-pair accumulators kept as 64-bit registers (no repacking inside the edge loop).
__device__ __forceinline__ uint64_t pk2(float x, float y) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& x, float& y) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ void ffma2p(uint64_t& acc, uint64_t a, uint64_t s2) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(s2));
}
__device__ __forceinline__ void fadd2p(uint64_t& acc, uint64_t a) {
    asm("add.rn.f32x2 %0, %1, %0;" : "+l"(acc) : "l"(a));
}
// acc2 (VN/2 pairs) += s * v (SCALED) or += v
template <typename T, bool SCALED> __device__ __forceinline__ void acc_vec2(uint64_t* acc2, const typename Vec<T>::raw& v, uint64_t s2);
template <> __device__ __forceinline__ void acc_vec2<float, true>(uint64_t* a, const float4& v, uint64_t s2) {
    ffma2p(a[0], pk2(v.x, v.y), s2);
    ffma2p(a[1], pk2(v.z, v.w), s2);
}
template <> __device__ __forceinline__ void acc_vec2<float, false>(uint64_t* a, const float4& v, uint64_t) {
    fadd2p(a[0], pk2(v.x, v.y));
    fadd2p(a[1], pk2(v.z, v.w));
}
template <> __device__ __forceinline__ void acc_vec2<__nv_bfloat16, true>(uint64_t* a, const uint4& v, uint64_t s2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) ffma2p(a[k], pk2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u)), s2);
}
// unscaled bf16: sm_100's mixed-precision add (add.rn.f32.bf16 -> FHADD.BF16) reads each bf16 half of the packed
// word directly (.H0 / .H1), one instruction per element instead of an unpack per element plus half an FADD2 --
// the same fp32 round-to-nearest sum of the exactly widened value, so the results are bitwise those of the unpacked
// FADD2 form
template <> __device__ __forceinline__ void acc_vec2<__nv_bfloat16, false>(uint64_t* a, const uint4& v, uint64_t) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float lo, hi;
        upk2(a[k], lo, hi);
        asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\tadd.rn.f32.bf16 %0, l, %0;\n\tadd.rn.f32.bf16 %1, h, %1;\n\t}"
            : "+f"(lo), "+f"(hi) : "r"(w[k]));
        a[k] = pk2(lo, hi);
    }
}

// acc (VN floats) += s * v, or += v when SCALED is false
template <typename T, bool SCALED> __device__ __forceinline__ void acc_vec(float* acc, const typename Vec<T>::raw& v, float s);
template <> __device__ __forceinline__ void acc_vec<float, true>(float* acc, const float4& v, float s) {
    ffma2(acc, v.x, v.y, s);
    ffma2(acc + 2, v.z, v.w, s);
}
template <> __device__ __forceinline__ void acc_vec<float, false>(float* acc, const float4& v, float) {
    fadd2(acc, v.x, v.y);
    fadd2(acc + 2, v.z, v.w);
}
template <> __device__ __forceinline__ void acc_vec<__nv_bfloat16, true>(float* acc, const uint4& v, float s) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) ffma2(acc + 2 * k, __uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u), s);
}
template <> __device__ __forceinline__ void acc_vec<__nv_bfloat16, false>(float* acc, const uint4& v, float) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) fadd2(acc + 2 * k, __uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u));
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

template <typename R> __device__ __forceinline__ R ldg_nc(const R* p) { return __ldg(p); }
#if defined(BNS_LDG_NA)
#define BNS_LDG_HINT ".L1::no_allocate"
#elif defined(BNS_LDG_EL)
#define BNS_LDG_HINT ".L1::evict_last"
#elif defined(BNS_LDG_EF)
#define BNS_LDG_HINT ".L1::evict_first"
#else
#define BNS_LDG_HINT ""
#endif
template <> __device__ __forceinline__ uint4 ldg_nc<uint4>(const uint4* p) {
    uint4 r;
    asm("ld.global.nc" BNS_LDG_HINT ".v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Philox4x32-10 (Salmon et al., SC'11), all four output words
__device__ __forceinline__ uint4 philox4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

}  // namespace bns
