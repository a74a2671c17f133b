// codec.cuh -- compute-weight codecs, bit-exact with the reference's
// quantize_value + pack_reduced (tensor.hpp:38-151) and unpack_reduced
// (tensor.hpp:153-183).
//
//  * width 2: IEEE binary16 round-to-nearest-even, overflow -> inf, binary16
//    subnormals honoured.  __float2half_rn is exactly that for every non-NaN
//    input (binary32 subnormal inputs round to +-0 either way); NaN encodes
//    as sign|0x7e00 (tensor.hpp:135-138), not the 0x7fff __float2half_rn gives.
//  * width 1: the reference's own E4M3 (bias 7, IEEE-style exponent 15 =
//    inf/NaN, SATURATING at 240 -- not OCP e4m3fn), so no cvt.e4m3 here.
//  * width 4: identity (fp32 bits).
#pragma once

#include <cuda_fp16.h>

#include "mlck_common.cuh"

namespace mlck {
namespace codec {

__device__ __forceinline__ uint16_t encode_half(float x) {
  const uint32_t bits = __float_as_uint(x);
  if ((bits & 0x7f800000u) == 0x7f800000u && (bits & 0x7fffffu))
    return static_cast<uint16_t>(((bits >> 16) & 0x8000u) | 0x7e00u);
  return __half_as_ushort(__float2half_rn(x));
}

__device__ __forceinline__ uint8_t encode_e4m3(float x) {
  const uint32_t bits = __float_as_uint(x);
  const uint32_t sign = (bits >> 24) & 0x80u;
  const int32_t exp = static_cast<int32_t>((bits >> 23) & 0xff) - 127;
  const uint32_t frac = bits & 0x7fffffu;
  if (exp == 128) return static_cast<uint8_t>(sign | 0x78u | (frac ? 0x4u : 0u));  // inf/nan
  if ((bits & 0x7fffffffu) == 0 || exp == -127) return static_cast<uint8_t>(sign);  // zero, fp32 subnormal
  const uint64_t mant = (1ull << 23) | frac;
  int shift = 20;
  if (exp < -6) shift += -6 - exp;
  if (shift >= 63) return static_cast<uint8_t>(sign);
  const uint64_t keep = mant >> shift;
  const uint64_t rem = mant & ((1ull << shift) - 1);
  const uint64_t half = 1ull << (shift - 1);
  uint64_t r = keep;
  if (rem > half || (rem == half && (keep & 1))) r += 1;
  if (exp < -6) return static_cast<uint8_t>(sign | static_cast<uint32_t>(r));  // subnormal grid (r <= 8)
  int32_t e = exp;
  if (r == 16) {
    r = 8;
    e += 1;
  }
  if (e > 7) return static_cast<uint8_t>(sign | 0x77u);  // saturate at 240
  return static_cast<uint8_t>(sign | (static_cast<uint32_t>(e + 7) << 3) | static_cast<uint32_t>(r - 8));
}

__device__ __forceinline__ float decode_half(uint16_t c) {
  // unpack_reduced(c, 5, 10) == IEEE half -> float widening (NaN payload kept)
  const uint32_t sign = static_cast<uint32_t>(c & 0x8000u) << 16;
  const uint32_t e = (c >> 10) & 0x1f, f = c & 0x3ffu;
  uint32_t bits;
  if (e == 0) {
    if (f == 0) {
      bits = sign;
    } else {
      int ee = -14;
      uint32_t m = f;
      while (!(m & 0x400u)) {
        m <<= 1;
        --ee;
      }
      bits = sign | (static_cast<uint32_t>(ee + 127) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (e == 0x1f) {
    bits = sign | 0x7f800000u | (f << 13);
  } else {
    bits = sign | ((e - 15 + 127) << 23) | (f << 13);
  }
  return __uint_as_float(bits);
}

__device__ __forceinline__ float decode_e4m3(uint8_t c) {
  const uint32_t sign = static_cast<uint32_t>(c & 0x80u) << 24;
  const uint32_t e = (c >> 3) & 0xf, f = c & 0x7u;
  uint32_t bits;
  if (e == 0) {
    if (f == 0) {
      bits = sign;
    } else {
      int ee = -6;
      uint32_t m = f;
      while (!(m & 0x8u)) {
        m <<= 1;
        --ee;
      }
      bits = sign | (static_cast<uint32_t>(ee + 127) << 23) | ((m & 0x7u) << 20);
    }
  } else if (e == 0xf) {
    bits = sign | 0x7f800000u | (f << 20);
  } else {
    bits = sign | ((e - 7 + 127) << 23) | (f << 20);
  }
  return __uint_as_float(bits);
}

// ---- generic reduced formats (ebits exponent, mbits mantissa bits, IEEE-
// style: exponent all-ones = inf/NaN), the reference's pack_reduced /
// unpack_reduced for any width (tensor.hpp:127-183).  x is expected on the
// target grid (it came out of quantize), so packing truncates; NaN keeps
// only the quiet bit, finite values above the format saturate to inf's code.
__device__ __forceinline__ uint16_t pack_generic(float x, int eb, int mb) {
  const uint32_t bits = __float_as_uint(x);
  const int bias = (1 << (eb - 1)) - 1;
  const uint32_t sign = (bits >> 31) << (eb + mb);
  const int e = static_cast<int>((bits >> 23) & 0xffu) - 127;
  const uint32_t frac = bits & 0x7fffffu, emask = (1u << eb) - 1u;
  if (e == 128) return static_cast<uint16_t>(sign | (emask << mb) | (frac ? 1u << (mb - 1) : 0u));
  if ((bits & 0x7fffffffu) == 0) return static_cast<uint16_t>(sign);
  if (e > bias) return static_cast<uint16_t>(sign | (emask << mb));
  const int emin = 1 - bias;
  if (e >= emin) return static_cast<uint16_t>(sign | (static_cast<uint32_t>(e + bias) << mb) | (frac >> (23 - mb)));
  const int sh = 23 - mb + (emin - e);  // subnormal of the target
  return static_cast<uint16_t>(sh > 31 ? sign : sign | (((1u << 23) | frac) >> sh));
}
__device__ __forceinline__ float unpack_generic(uint16_t c, int eb, int mb) {
  const int bias = (1 << (eb - 1)) - 1;
  const uint32_t emask = (1u << eb) - 1u, fmask = (1u << mb) - 1u;
  const uint32_t sign = (static_cast<uint32_t>(c) >> (eb + mb)) << 31;
  const uint32_t e = (c >> mb) & emask, f = c & fmask;
  uint32_t bits;
  if (e == 0) {
    if (f == 0) {
      bits = sign;
    } else {  // normalise the subnormal
      int ee = 1 - bias;
      uint32_t m = f;
      while (!(m & (1u << mb))) {
        m <<= 1;
        --ee;
      }
      bits = sign | (static_cast<uint32_t>(ee + 127) << 23) | ((m & fmask) << (23 - mb));
    }
  } else if (e == emask) {
    bits = sign | 0x7f800000u | (f << (23 - mb));
  } else {
    bits = sign | (static_cast<uint32_t>(static_cast<int>(e) - bias + 127) << 23) | (f << (23 - mb));
  }
  return __uint_as_float(bits);
}

// Writes the code of x at element i of a code array of width cb.
__device__ __forceinline__ void store_code(void* codes, uint64_t i, float x, int cb) {
  if (cb == 2) static_cast<uint16_t*>(codes)[i] = encode_half(x);
  else if (cb == 1) static_cast<uint8_t*>(codes)[i] = encode_e4m3(x);
  else static_cast<float*>(codes)[i] = x;
}
__device__ __forceinline__ float load_code(const void* codes, uint64_t i, int cb) {
  if (cb == 2) return decode_half(static_cast<const uint16_t*>(codes)[i]);
  if (cb == 1) return decode_e4m3(static_cast<const uint8_t*>(codes)[i]);
  return static_cast<const float*>(codes)[i];
}

}  // namespace codec
}  // namespace mlck
