/*
 * moelab_oracle.c -- CPU restatement of the reference checkpoint data path.
 *
 * TEST INFRASTRUCTURE ONLY (see moelab_oracle.h).  Parity of this file is
 * pinned against the real reference compiled into oracle/_ref
 * (tests/test_oracle.py) and against tests/golden/.
 *
 * Citations are /root/reference/proj/include/moelab/<file>:<line>.
 */
#include "moelab_oracle.h"

#include <math.h>
#include <string.h>

/* ---- digest.hpp:18-25 ------------------------------------------------- */
uint64_t mlo_fnv1a64(const uint8_t* data, size_t n, uint64_t seed) {
  uint64_t h = seed;
  for (size_t i = 0; i < n; ++i) {
    h ^= data[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* ---- tensor.hpp:38-92 round_to_format --------------------------------- */
static float round_to_format(float x, int ebits, int mbits, int saturate) {
  if (isnan(x) || isinf(x)) return x;
  uint32_t bits;
  memcpy(&bits, &x, 4);
  const uint32_t sign = bits & 0x80000000u;
  int32_t exp = (int32_t)((bits >> 23) & 0xff) - 127;
  uint32_t frac = bits & 0x7fffffu;
  if ((bits & 0x7fffffffu) == 0) return x; /* signed zero */
  const int bias = (1 << (ebits - 1)) - 1;
  const int emax = bias;
  const int emin = 1 - bias;
  if (exp == -127) { /* binary32 subnormal: flush to signed zero */
    float z;
    memcpy(&z, &sign, 4);
    return z;
  }
  uint64_t mant = (1ull << 23) | frac;
  int shift = 23 - mbits;
  if (exp < emin) shift += emin - exp;
  if (shift >= 63) {
    float z;
    memcpy(&z, &sign, 4);
    return z;
  }
  const uint64_t keep = mant >> shift;
  const uint64_t rem = mant & ((1ull << shift) - 1);
  const uint64_t half = 1ull << (shift - 1);
  uint64_t rounded = keep;
  if (rem > half || (rem == half && (keep & 1))) rounded += 1;
  double mag = ldexp((double)rounded, exp - 23 + shift);
  const double max_finite = ldexp((double)((2 << mbits) - 1), emax - mbits);
  if (mag > max_finite) {
    if (saturate) {
      mag = max_finite;
    } else {
      return sign ? -INFINITY : INFINITY;
    }
  }
  float out = (float)mag;
  return sign ? -out : out;
}

/* ---- tensor.hpp:99-111 quantize_value --------------------------------- */
int mlo_quantize_value(float x, int compute_bytes, float* out) {
  switch (compute_bytes) {
    case 4: *out = x; return 0;
    case 2: *out = round_to_format(x, 5, 10, 0); return 0;
    case 1: *out = round_to_format(x, 4, 3, 1); return 0;
    default: return -1;
  }
}

int mlo_quantize_array(const float* in, size_t n, int compute_bytes, float* out) {
  for (size_t i = 0; i < n; ++i)
    if (mlo_quantize_value(in[i], compute_bytes, out + i) != 0) return -1;
  return 0;
}

/* ---- tensor.hpp:127-151 pack_reduced ---------------------------------- */
uint16_t mlo_pack_reduced(float x, int ebits, int mbits) {
  uint32_t bits;
  memcpy(&bits, &x, 4);
  const int bias = (1 << (ebits - 1)) - 1;
  const uint16_t sign = (uint16_t)((bits >> 31) << (ebits + mbits));
  int32_t exp = (int32_t)((bits >> 23) & 0xff) - 127;
  uint32_t frac = bits & 0x7fffffu;
  const uint32_t exp_mask = (1u << ebits) - 1;
  if (exp == 128) return (uint16_t)(sign | (exp_mask << mbits) | (frac ? (1u << (mbits - 1)) : 0));
  if ((bits & 0x7fffffffu) == 0) return sign;
  if (exp > bias) return (uint16_t)(sign | (exp_mask << mbits));
  const int emin = 1 - bias;
  if (exp >= emin) return (uint16_t)(sign | ((uint32_t)(exp + bias) << mbits) | (frac >> (23 - mbits)));
  uint32_t mant = (1u << 23) | frac;
  int shift = (23 - mbits) + (emin - exp);
  if (shift > 31) return sign;
  return (uint16_t)(sign | (mant >> shift));
}

/* ---- tensor.hpp:153-183 unpack_reduced -------------------------------- */
float mlo_unpack_reduced(uint16_t code, int ebits, int mbits) {
  const int bias = (1 << (ebits - 1)) - 1;
  const uint32_t exp_mask = (1u << ebits) - 1;
  const uint32_t frac_mask = (1u << mbits) - 1;
  const uint32_t sign = ((uint32_t)code >> (ebits + mbits)) << 31;
  const uint32_t exp = (code >> mbits) & exp_mask;
  const uint32_t frac = code & frac_mask;
  uint32_t bits;
  if (exp == 0) {
    if (frac == 0) {
      bits = sign;
    } else {
      int e = 1 - bias;
      uint32_t m = frac;
      while (!(m & (1u << mbits))) {
        m <<= 1;
        --e;
      }
      m &= frac_mask;
      bits = sign | ((uint32_t)(e + 127) << 23) | (m << (23 - mbits));
    }
  } else if (exp == exp_mask) {
    bits = sign | 0x7f800000u | (frac << (23 - mbits));
  } else {
    bits = sign | ((uint32_t)((int32_t)exp - bias + 127) << 23) | (frac << (23 - mbits));
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

/* ---- snapshot.hpp:77-111 write_compute / read_compute ------------------ */
int64_t mlo_encode_compute(const float* vals, size_t n, int compute_bytes, uint8_t* out) {
  switch (compute_bytes) {
    case 4: memcpy(out, vals, n * 4); return (int64_t)(n * 4);
    case 2:
      for (size_t i = 0; i < n; ++i) {
        uint16_t c = mlo_pack_reduced(vals[i], 5, 10);
        memcpy(out + 2 * i, &c, 2);
      }
      return (int64_t)(n * 2);
    case 1:
      for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)mlo_pack_reduced(vals[i], 4, 3);
      return (int64_t)n;
    default: return -1;
  }
}

int64_t mlo_decode_compute(const uint8_t* in, size_t n, int compute_bytes, float* vals) {
  switch (compute_bytes) {
    case 4: memcpy(vals, in, n * 4); return (int64_t)(n * 4);
    case 2:
      for (size_t i = 0; i < n; ++i) {
        uint16_t c;
        memcpy(&c, in + 2 * i, 2);
        vals[i] = mlo_unpack_reduced(c, 5, 10);
      }
      return (int64_t)(n * 2);
    case 1:
      for (size_t i = 0; i < n; ++i) vals[i] = mlo_unpack_reduced(in[i], 4, 3);
      return (int64_t)n;
    default: return -1;
  }
}

/* ---- snapshot.hpp:61-73 container layout ------------------------------- */
#define MLO_MAGIC 0x4b434c4du
#define MLO_VERSION 1u
#define MLO_HEADER_BYTES 45u
#define MLO_ENTRY_HEADER_BYTES 13u

uint64_t mlo_record_size(const mlo_entry* e, size_t n, int compute_bytes) {
  uint64_t s = MLO_HEADER_BYTES;
  for (size_t i = 0; i < n; ++i) {
    s += MLO_ENTRY_HEADER_BYTES;
    if (e[i].mode == 0) s += 8 + 12 * e[i].param_count;
    else s += (uint64_t)compute_bytes * e[i].param_count;
  }
  return s + 8;
}

#define PUT(T, val)            \
  do {                         \
    T _v = (T)(val);           \
    memcpy(out + pos, &_v, sizeof(T)); \
    pos += sizeof(T);          \
  } while (0)

/* ---- snapshot.hpp:115-144 serialize_record ----------------------------- */
int64_t mlo_serialize_record(const mlo_header* h, const mlo_entry* e, size_t n,
                             int compute_bytes, uint8_t* out) {
  if (compute_bytes != 1 && compute_bytes != 2 && compute_bytes != 4) return -1;
  uint64_t pos = 0;
  PUT(uint32_t, MLO_MAGIC);
  PUT(uint32_t, MLO_VERSION);
  PUT(uint8_t, h->kind);
  PUT(uint64_t, h->iteration);
  PUT(uint64_t, h->window_start);
  PUT(uint32_t, h->wsparse);
  PUT(uint32_t, h->slot);
  PUT(uint64_t, h->data_seed);
  PUT(uint32_t, (uint32_t)n);
  for (size_t i = 0; i < n; ++i) {
    PUT(uint32_t, e[i].id);
    PUT(uint8_t, e[i].mode);
    PUT(uint64_t, e[i].param_count);
    const size_t P = (size_t)e[i].param_count;
    if (e[i].mode == 0) {
      PUT(uint64_t, e[i].step);
      memcpy(out + pos, e[i].master, P * 4); pos += P * 4;
      memcpy(out + pos, e[i].m, P * 4); pos += P * 4;
      memcpy(out + pos, e[i].v, P * 4); pos += P * 4;
    } else {
      pos += (uint64_t)mlo_encode_compute(e[i].compute, P, compute_bytes, out + pos);
    }
  }
  const uint64_t sum = mlo_fnv1a64(out, pos, 0xcbf29ce484222325ull);
  PUT(uint64_t, sum);
  return (int64_t)pos;
}

const char* mlo_error_text(int code) {
  switch (code) {
    case MLO_OK: return "";
    case MLO_E_TRUNCATED: return "container truncated";
    case MLO_E_CHECKSUM: return "container checksum mismatch";
    case MLO_E_MAGIC: return "container: bad magic";
    case MLO_E_VERSION: return "container: unsupported version";
    case MLO_E_WIDTH: return "container: unsupported compute width";
    default: return "unknown error";
  }
}

/* ---- snapshot.hpp:153-197 parse_record --------------------------------- */
int mlo_parse_record(const uint8_t* blob, uint64_t n, int compute_bytes, mlo_header* h,
                     uint32_t* n_entries, mlo_parsed_entry* entries, uint32_t max_entries,
                     uint32_t* version_out) {
  if (n < 8) return MLO_E_TRUNCATED;
  uint64_t trailer;
  memcpy(&trailer, blob + n - 8, 8);
  if (trailer != mlo_fnv1a64(blob, n - 8, 0xcbf29ce484222325ull)) return MLO_E_CHECKSUM;
  const uint64_t end = n - 8;
  uint64_t pos = 0;
#define GET(T, dst)                                  \
  do {                                               \
    if (pos + sizeof(T) > end) return MLO_E_TRUNCATED; \
    memcpy(&(dst), blob + pos, sizeof(T));           \
    pos += sizeof(T);                                \
  } while (0)
  uint32_t magic, version, count;
  GET(uint32_t, magic);
  if (magic != MLO_MAGIC) return MLO_E_MAGIC;
  GET(uint32_t, version);
  if (version_out) *version_out = version;
  if (version != MLO_VERSION) return MLO_E_VERSION;
  GET(uint8_t, h->kind);
  GET(uint64_t, h->iteration);
  GET(uint64_t, h->window_start);
  GET(uint32_t, h->wsparse);
  GET(uint32_t, h->slot);
  GET(uint64_t, h->data_seed);
  GET(uint32_t, count);
  *n_entries = count;
  for (uint32_t i = 0; i < count; ++i) {
    mlo_parsed_entry pe;
    GET(uint32_t, pe.id);
    GET(uint8_t, pe.mode);
    GET(uint64_t, pe.param_count);
    pe.step = 0;
    if (pe.mode == 0) {
      GET(uint64_t, pe.step);
      pe.payload_offset = pos;
      const uint64_t need = 12 * pe.param_count;
      if (pe.param_count > end || pos + need > end) return MLO_E_TRUNCATED;
      pos += need;
    } else {
      if (compute_bytes != 1 && compute_bytes != 2 && compute_bytes != 4) return MLO_E_WIDTH;
      pe.payload_offset = pos;
      const uint64_t need = (uint64_t)compute_bytes * pe.param_count;
      if (pe.param_count > end || pos + need > end) return MLO_E_TRUNCATED;
      pos += need;
    }
    if (i < max_entries) entries[i] = pe;
  }
#undef GET
  return MLO_OK;
}

/* ---- engine.hpp:738-753 optimizer_step_adam ---------------------------- */
float mlo_bias_correction(float beta, uint64_t step) {
  return 1.0f - powf(beta, (float)step);
}

void mlo_adam_step(float* master, float* m, float* v, uint64_t* step, const float* grad,
                   size_t n, float lr, float beta1, float beta2, float eps) {
  *step += 1;
  const float bc1 = 1.0f - powf(beta1, (float)*step);
  const float bc2 = 1.0f - powf(beta2, (float)*step);
  const float omb1 = 1.0f - beta1;
  const float omb2 = 1.0f - beta2;
  for (size_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + omb1 * grad[i];
    v[i] = beta2 * v[i] + omb2 * grad[i] * grad[i];
    master[i] -= lr * (m[i] / bc1) / (sqrtf(v[i] / bc2) + eps);
  }
}

/* ---- engine.hpp:710-713 SGD branch ------------------------------------- */
void mlo_sgd_step(float* master, uint64_t* step, const float* grad, size_t n, float lr) {
  for (size_t i = 0; i < n; ++i) master[i] -= lr * grad[i];
  *step += 1;
}

void mlo_replay_op(float* master, float* m, float* v, uint64_t* step, const float* grads,
                   uint32_t n_steps, size_t n, int optimizer_kind, float lr, float beta1,
                   float beta2, float eps) {
  for (uint32_t s = 0; s < n_steps; ++s) {
    if (optimizer_kind == 0)
      mlo_adam_step(master, m, v, step, grads + (size_t)s * n, n, lr, beta1, beta2, eps);
    else
      mlo_sgd_step(master, step, grads + (size_t)s * n, n, lr);
  }
}

/* ---- engine.hpp:246-261 serialize_state ("MLST") ----------------------- */
uint64_t mlo_state_size(const mlo_state_op* ops, size_t n_ops) {
  uint64_t s = 4 + 4 + 8 + 8 + 4;
  for (size_t i = 0; i < n_ops; ++i) s += 16 + 12 * ops[i].param_count;
  return s;
}

uint64_t mlo_serialize_state(uint64_t iteration, uint64_t data_seed, const mlo_state_op* ops,
                             size_t n_ops, uint8_t* out) {
  uint64_t pos = 0;
  PUT(uint32_t, 0x4d4c5354u);
  PUT(uint32_t, 1u);
  PUT(uint64_t, iteration);
  PUT(uint64_t, data_seed);
  PUT(uint32_t, (uint32_t)n_ops);
  for (size_t i = 0; i < n_ops; ++i) {
    const size_t P = (size_t)ops[i].param_count;
    PUT(uint64_t, ops[i].step);
    PUT(uint64_t, ops[i].param_count);
    if (P) {
      memcpy(out + pos, ops[i].master, P * 4); pos += P * 4;
      memcpy(out + pos, ops[i].m, P * 4); pos += P * 4;
      memcpy(out + pos, ops[i].v, P * 4); pos += P * 4;
    }
  }
  return pos;
}
#undef PUT

/* ---- rng.hpp:15-32, 35-38, 85-96 --------------------------------------- */
static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9e3779b97f4a7c15ull;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void mlo_rng_seed(mlo_rng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
}

uint64_t mlo_rng_next(mlo_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

double mlo_rng_uniform(mlo_rng* r) { return (double)(mlo_rng_next(r) >> 11) * 0x1.0p-53; }
double mlo_rng_uniform_range(mlo_rng* r, double lo, double hi) {
  return lo + (hi - lo) * mlo_rng_uniform(r);
}

void mlo_rng_substream(const mlo_rng* r, const char* label, uint64_t index, mlo_rng* out) {
  uint64_t h = 0xcbf29ce484222325ull;
#define MIX(val)               \
  do {                         \
    h ^= (uint64_t)(val);      \
    h *= 0x100000001b3ull;     \
  } while (0)
  for (const char* c = label; *c; ++c) MIX((uint8_t)*c);
  MIX(index);
  MIX(r->s[0]);
  MIX(r->s[2]);
#undef MIX
  mlo_rng_seed(out, h);
}

/* ---- engine.hpp:283-296 init_state master draw ------------------------- */
void mlo_init_master(uint64_t seed, uint32_t op_id, int32_t token_dim, float* master, size_t n) {
  mlo_rng root, r;
  mlo_rng_seed(&root, seed);
  mlo_rng_substream(&root, "init", op_id, &r);
  const double scale = 0.5 / sqrt((double)token_dim);
  for (size_t i = 0; i < n; ++i) master[i] = (float)mlo_rng_uniform_range(&r, -scale, scale);
}

/* ---- counter-based synthetic generator (benchmark inputs) -------------- */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

float mlo_synth_value(uint64_t seed, uint64_t stream, uint64_t index, float lo, float hi) {
  const uint64_t key = mix64(seed + 0x632be59bd9b4e019ull * (stream + 1));
  const uint64_t x = mix64(key ^ index);
  const float u = (float)(x >> 40) * 0x1.0p-24f;
  const float span = hi - lo;
  const float t = span * u;
  return lo + t;
}

void mlo_synth_fill(uint64_t seed, uint64_t stream, float lo, float hi, float* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = mlo_synth_value(seed, stream, i, lo, hi);
}

/* elements [first, first + n) of the stream (chunked checks of big operators) */
void mlo_synth_fill_range(uint64_t seed, uint64_t stream, float lo, float hi, float* out, uint64_t first,
                          size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = mlo_synth_value(seed, stream, first + i, lo, hi);
}
