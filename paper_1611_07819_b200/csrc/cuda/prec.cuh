// SPDX-License-Identifier: Apache-2.0
// Device-side storage codec shared by the HBM-bound kernels: load an element
// of any storage precision into the compute type, store back with the
// reference's rounding (proj/include/gridmath/precision.hpp:42-149):
// any -> Half rounds through float (RNE, >= 65520 -> inf, NaN payload kept),
// Double -> Single RNE, BF16 (new tag 3) RNE from float. Half is widened
// IEEE-exactly (the reference halves subnormals).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace gmk {

__device__ __forceinline__ uint16_t f32_to_half_bits(float f) {
  const uint32_t x = __float_as_uint(f);
  if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x007FFFFFu) != 0) {
    // NaN: sign, all-ones exponent, payload = top 10 mantissa bits (never 0).
    uint32_t pay = (x & 0x007FFFFFu) >> 13;
    if (pay == 0) pay = 1;
    return static_cast<uint16_t>(((x >> 16) & 0x8000u) | 0x7C00u | pay);
  }
  // Finite and inf: IEEE binary16 RNE (overflow -> inf) is exactly the
  // reference's hand-rolled rounding.
  return __half_as_ushort(__float2half_rn(f));
}

__device__ __forceinline__ float half_bits_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  const uint32_t m = h & 0x3FFu;
  if (e == 31) return __uint_as_float(sign | 0x7F800000u | (m << 13));  // inf / NaN payload kept
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ double load_elem(const void* base, int prec, uint64_t idx) {
  switch (prec) {
    case 0: return static_cast<double>(half_bits_to_f32(reinterpret_cast<const uint16_t*>(base)[idx]));
    case 1: return static_cast<double>(reinterpret_cast<const float*>(base)[idx]);
    case 2: return reinterpret_cast<const double*>(base)[idx];
    default: {
      const uint32_t b = static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(base)[idx]) << 16;
      return static_cast<double>(__uint_as_float(b));
    }
  }
}

__device__ __forceinline__ float load_elem_f32(const void* base, int prec, uint64_t idx) {
  switch (prec) {
    case 0: return half_bits_to_f32(reinterpret_cast<const uint16_t*>(base)[idx]);
    case 1: return reinterpret_cast<const float*>(base)[idx];
    case 2: return static_cast<float>(reinterpret_cast<const double*>(base)[idx]);
    default: return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(base)[idx]) << 16);
  }
}

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__device__ __forceinline__ void store_elem(void* base, int prec, uint64_t idx, double v) {
  switch (prec) {
    case 0: reinterpret_cast<uint16_t*>(base)[idx] = f32_to_half_bits(__double2float_rn(v)); break;
    case 1: reinterpret_cast<float*>(base)[idx] = __double2float_rn(v); break;
    case 2: reinterpret_cast<double*>(base)[idx] = v; break;
    default: reinterpret_cast<uint16_t*>(base)[idx] = f32_to_bf16_bits(__double2float_rn(v)); break;
  }
}

__device__ __forceinline__ void store_elem_f32(void* base, int prec, uint64_t idx, float v) {
  switch (prec) {
    case 0: reinterpret_cast<uint16_t*>(base)[idx] = f32_to_half_bits(v); break;
    case 1: reinterpret_cast<float*>(base)[idx] = v; break;
    case 2: reinterpret_cast<double*>(base)[idx] = static_cast<double>(v); break;
    default: reinterpret_cast<uint16_t*>(base)[idx] = f32_to_bf16_bits(v); break;
  }
}

}  // namespace gmk

namespace gmk {

// Compute-type views of the codec: T = float (Single compute) or double
// (Double compute), the reference's loadScalar<T>/storeScalar<T>.
template <typename T>
__device__ __forceinline__ T load_as(const void* base, int prec, uint64_t idx);
template <>
__device__ __forceinline__ float load_as<float>(const void* base, int prec, uint64_t idx) {
  return load_elem_f32(base, prec, idx);
}
template <>
__device__ __forceinline__ double load_as<double>(const void* base, int prec, uint64_t idx) {
  return load_elem(base, prec, idx);
}
__device__ __forceinline__ void store_as(void* base, int prec, uint64_t idx, float v) { store_elem_f32(base, prec, idx, v); }
__device__ __forceinline__ void store_as(void* base, int prec, uint64_t idx, double v) { store_elem(base, prec, idx, v); }

// Separately rounded multiply / add: the reference is built without FMA
// contraction, and nvcc would otherwise fuse a*b+c.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

}  // namespace gmk
