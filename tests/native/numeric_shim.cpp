// Host build of the kernels' bit-level numerics (paper_2506_11277_b200/csrc/
// ozgpu_numeric.h) for CPU unit tests: the same source the GPU runs.
#include <cstdint>

#include "ozgpu_numeric.h"

using namespace ozgpu;

extern "C" {
double nt_ldexp_rn(double d, long e) { return ldexp_rn(d, e); }

// v (words little-endian, W = 2 or 3) accumulated from (s_i << shift_i), then rounded
double nt_accumulate_round(int words, int n, const int32_t* s, const int* shift, long e) {
  if (words == 2) {
    uint64_t v[2] = {0, 0};
    for (int i = 0; i < n; ++i) words_add_shifted<2>(v, s[i], shift[i]);
    return round_words<2>(v, e);
  }
  if (words == 3) {
    uint64_t v[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) words_add_shifted<3>(v, s[i], shift[i]);
    return round_words<3>(v, e);
  }
  uint64_t v[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) words_add_shifted<6>(v, s[i], shift[i]);
  return round_words<6>(v, e);
}

void nt_accumulate_words(int n, const int32_t* s, const int* shift, uint64_t* out6) {
  uint64_t v[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) words_add_shifted<6>(v, s[i], shift[i]);
  for (int w = 0; w < 6; ++w) out6[w] = v[w];
}

void nt_slices(double x, int q, int width, int count, int mode, long long* out) {
  SliceEntry e = make_slice_entry(x, q, width, count, mode);
  for (int l = 0; l < count; ++l) out[l] = slice_of(e, l, width, count, mode);
}
}

extern "C" double nt_round_i128(uint64_t lo, uint64_t hi, long e) {
  unsigned __int128 v = (static_cast<unsigned __int128>(hi) << 64) | lo;
  return round_i128(v, e);
}

extern "C" double nt_round_hilo(uint64_t lo, uint64_t hi, long e) { return round_hilo(hi, lo, e); }

extern "C" double nt_round_w3(uint64_t w0, uint64_t w1, uint64_t w2, long e) {
  return round_w3(w2, w1, w0, e);
}
