// elem.cuh -- storage types of the joint tensor (logits in, grads out): fp32, fp16, bf16.  All arithmetic is
// fp32 (and fp64 in K2); 16-bit storage only changes how a 128-bit vector is unpacked and packed.
// PAPER.md §4.2 P:161 ("populate the lattice with a half (fp16) precision tensor and cast it to fp32 or fp64
// only for the forward-backward score calculation").
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rnnt {

enum Dtype : int { kF32 = 0, kF16 = 1, kBF16 = 2 };

inline size_t dtype_size(int dt) { return dt == kF32 ? 4 : 2; }

template <typename T>
struct Elem;

template <>
struct Elem<float> {
    static constexpr int kPerVec = 4;  // elements per 128-bit vector
    __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[4]) {
        f[0] = __uint_as_float(v.x);
        f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z);
        f[3] = __uint_as_float(v.w);
    }
    __device__ __forceinline__ static uint4 pack(const float (&f)[4]) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                          __float_as_uint(f[3]));
    }
    // 64-bit vectors (2 elements): rows whose length is even but not a multiple of 4
    __device__ __forceinline__ static void unpack(const uint2& v, float (&f)[2]) {
        f[0] = __uint_as_float(v.x);
        f[1] = __uint_as_float(v.y);
    }
    __device__ __forceinline__ static uint2 pack(const float (&f)[2]) {
        return make_uint2(__float_as_uint(f[0]), __float_as_uint(f[1]));
    }
    __device__ __forceinline__ static float to_f32(float x) { return x; }
    __device__ __forceinline__ static float from_f32(float x) { return x; }
};

template <>
struct Elem<__nv_bfloat16> {
    static constexpr int kPerVec = 8;
    __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // bf16 is the top half of an fp32: exact widening by a shift / mask
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    __device__ __forceinline__ static uint4 pack(const float (&f)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);  // round to nearest even
            w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
    // 64-bit vectors (4 elements): rows whose length is a multiple of 4 but not of 8 (e.g. V = 500)
    __device__ __forceinline__ static void unpack(const uint2& v, float (&f)[4]) {
        f[0] = __uint_as_float(v.x << 16);
        f[1] = __uint_as_float(v.x & 0xffff0000u);
        f[2] = __uint_as_float(v.y << 16);
        f[3] = __uint_as_float(v.y & 0xffff0000u);
    }
    __device__ __forceinline__ static uint2 pack(const float (&f)[4]) {
        const __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]), b = __floats2bfloat162_rn(f[2], f[3]);
        return make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
    __device__ __forceinline__ static float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
    __device__ __forceinline__ static __nv_bfloat16 from_f32(float x) { return __float2bfloat16_rn(x); }
};

template <>
struct Elem<__half> {
    static constexpr int kPerVec = 8;
    __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 p = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            f[2 * i] = p.x;
            f[2 * i + 1] = p.y;
        }
    }
    __device__ __forceinline__ static uint4 pack(const float (&f)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
            w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
    __device__ __forceinline__ static void unpack(const uint2& v, float (&f)[4]) {
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
        f[0] = a.x;
        f[1] = a.y;
        f[2] = b.x;
        f[3] = b.y;
    }
    __device__ __forceinline__ static uint2 pack(const float (&f)[4]) {
        const __half2 a = __floats2half2_rn(f[0], f[1]), b = __floats2half2_rn(f[2], f[3]);
        return make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
    __device__ __forceinline__ static float to_f32(__half x) { return __half2float(x); }
    __device__ __forceinline__ static __half from_f32(float x) { return __float2half_rn(x); }
};

// 128-bit streaming accesses (see common.cuh for the policies).
__device__ __forceinline__ uint4 ldv_ro(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ldv(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol)
                 : "memory");
    return v;
}
__device__ __forceinline__ void stv(uint4* p, const uint4& v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}
// 64-bit variants (16-bit rows with V % 8 == 4)
__device__ __forceinline__ uint2 ldv_ro(const uint2* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ldv(const uint2* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol)
                 : "memory");
    return v;
}
__device__ __forceinline__ void stv(uint2* p, const uint2& v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "l"(pol)
                 : "memory");
}
template <typename VecT>
__device__ __forceinline__ VecT zero_vec();
template <>
__device__ __forceinline__ uint4 zero_vec<uint4>() { return make_uint4(0u, 0u, 0u, 0u); }
template <>
__device__ __forceinline__ uint2 zero_vec<uint2>() { return make_uint2(0u, 0u); }

// A vector of -inf in storage type Z (fills the slots past V without a per-element select)
template <typename Z> struct NegInfWord;
template <> struct NegInfWord<float> { static constexpr uint32_t kWord = 0xff800000u; };
template <> struct NegInfWord<__nv_bfloat16> { static constexpr uint32_t kWord = 0xff80ff80u; };
template <> struct NegInfWord<__half> { static constexpr uint32_t kWord = 0xfc00fc00u; };
template <typename Z, typename VecT>
__device__ __forceinline__ VecT neg_inf_vec() {
    constexpr uint32_t w = NegInfWord<Z>::kWord;
    if constexpr (sizeof(VecT) == 16)
        return make_uint4(w, w, w, w);
    else
        return make_uint2(w, w);
}

template <typename T>
__device__ __forceinline__ float lds_scalar(const T* p) {  // scalar read-only load, widened to fp32
    return Elem<T>::to_f32(__ldg(p));
}

}  // namespace rnnt
