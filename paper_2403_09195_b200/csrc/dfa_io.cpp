// DTNSR1 tensor files (the reference's golden-vector / dataset format,
// tensor_io.hpp:15-19, 52-156), host-side C-ABI:
//   magic "DTNSR1" | dtype byte (0 = f32, 1 = f64) | rank byte (<= 8) |
//   rank x uint32 little-endian dims | raw little-endian scalars, row-major.
// Errors map to DFA_ERR_IO (attnkit::io_error) with the reference's message
// text, so golden vectors written by either side load on the other.
#include <algorithm>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/dfa.h"

namespace dfa_impl {
dfa_status_t fail_msg(dfa_status_t st, const char* fmt, ...);  // dfa_api.cpp: sets dfa_last_error()
}
#define dfa_io_fail(...) dfa_impl::fail_msg(DFA_ERR_IO, __VA_ARGS__)

namespace {

constexpr char kMagic[6] = {'D', 'T', 'N', 'S', 'R', '1'};
constexpr int kMaxRank = 8;  // tensor_io.hpp:20

bool little_endian() {
  const uint16_t probe = 0x0102;
  uint8_t b;
  memcpy(&b, &probe, 1);
  return b == 0x02;
}

void swap_bytes(void* p, size_t width, size_t count) {
  auto* c = static_cast<uint8_t*>(p);
  for (size_t i = 0; i < count; ++i, c += width)
    for (size_t a = 0, b = width - 1; a < b; ++a, --b) {
      const uint8_t t = c[a];
      c[a] = c[b];
      c[b] = t;
    }
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

// tensor_io.hpp:97-118 read_tensor_header
dfa_status_t read_header(FILE* f, const char* path, int32_t* dtype, int32_t* rank, int64_t* dims) {
  char magic[6];
  uint8_t code = 0, rk = 0;
  auto truncated = [&] { return dfa_io_fail("truncated tensor file: %s", path); };
  if (fread(magic, 1, 6, f) != 6) return truncated();
  if (memcmp(magic, kMagic, 6) != 0) return dfa_io_fail("bad magic in tensor file: %s", path);
  if (fread(&code, 1, 1, f) != 1 || fread(&rk, 1, 1, f) != 1) return truncated();
  if (code > 1) return dfa_io_fail("unknown dtype code %d in %s", (int)code, path);
  if (rk > kMaxRank) return dfa_io_fail("rank %d exceeds format limit in %s", (int)rk, path);
  for (int i = 0; i < rk; ++i) {
    uint32_t d;
    if (fread(&d, 4, 1, f) != 1) return truncated();
    if (!little_endian()) swap_bytes(&d, 4, 1);
    dims[i] = (int64_t)d;
  }
  *dtype = code;
  *rank = rk;
  return DFA_OK;
}

}  // namespace

extern "C" {

dfa_status_t dfa_tensor_header(const char* path, int32_t* dtype, int32_t* rank, int64_t* dims) {
  if (!path || !dtype || !rank || !dims) return dfa_io_fail("dfa_tensor_header: null argument");
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return dfa_io_fail("cannot open tensor file: %s", path);
  return read_header(fh.f, path, dtype, rank, dims);
}

// tensor_io.hpp:147-153 load_tensor<Scalar>: the payload is converted to
// `want` (0 = f32, 1 = f64) like read_payload's cast (:122-144).
dfa_status_t dfa_tensor_load(const char* path, int32_t want, void* out, int64_t capacity) {
  if (!path || !out) return dfa_io_fail("dfa_tensor_load: null argument");
  if (want != 0 && want != 1) return dfa_io_fail("dfa_tensor_load: unknown dtype code %d", (int)want);
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return dfa_io_fail("cannot open tensor file: %s", path);
  int32_t dtype = 0, rank = 0;
  int64_t dims[kMaxRank];
  dfa_status_t st = read_header(fh.f, path, &dtype, &rank, dims);
  if (st != DFA_OK) return st;
  // Element count with an overflow check: a crafted header (up to 8 dims of
  // 2^32 - 1) must fail as io_error before anything is allocated or read.
  const size_t width = dtype == 0 ? 4 : 8;
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) {
    if (dims[i] != 0 && n > (int64_t)(SIZE_MAX / width) / dims[i])
      return dfa_io_fail("tensor file %s: element count overflows", path);
    n *= dims[i];
  }
  if (n > capacity) return dfa_io_fail("dfa_tensor_load: %s holds %lld scalars, buffer has %lld", path, (long long)n,
                                       (long long)capacity);
  if (dtype == want) {  // straight into the caller's buffer (sized above)
    if (n && fread(out, width, (size_t)n, fh.f) != (size_t)n) return dfa_io_fail("truncated tensor file: %s", path);
    if (!little_endian()) swap_bytes(out, width, (size_t)n);
    return DFA_OK;
  }
  // converting load: stream the payload through a bounded chunk buffer
  constexpr size_t kChunk = 1 << 14;
  std::vector<uint8_t> buf(kChunk * width);
  uint8_t* raw = buf.data();
  for (int64_t i0 = 0; i0 < n; i0 += (int64_t)kChunk) {
    const size_t c = (size_t)std::min<int64_t>((int64_t)kChunk, n - i0);
    if (fread(raw, width, c, fh.f) != c) return dfa_io_fail("truncated tensor file: %s", path);
    if (!little_endian()) swap_bytes(raw, width, c);
    if (dtype == 0) {
      const float* src = reinterpret_cast<const float*>(raw);
      double* dst = static_cast<double*>(out) + i0;
      for (size_t i = 0; i < c; ++i) dst[i] = (double)src[i];
    } else {
      const double* src = reinterpret_cast<const double*>(raw);
      float* dst = static_cast<float*>(out) + i0;
      for (size_t i = 0; i < c; ++i) dst[i] = (float)src[i];
    }
  }
  return DFA_OK;
}

// tensor_io.hpp:52-95 write_tensor / save_tensor
dfa_status_t dfa_tensor_save(const char* path, int32_t dtype, int32_t rank, const int64_t* dims, const void* data) {
  if (!path || (rank > 0 && !dims)) return dfa_io_fail("dfa_tensor_save: null argument");
  if (dtype != 0 && dtype != 1) return dfa_io_fail("dfa_tensor_save: unknown dtype code %d", (int)dtype);
  if (rank < 0 || rank > kMaxRank) return dfa_io_fail("tensor rank %d exceeds format limit %d", (int)rank, kMaxRank);
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) {
    if (dims[i] < 0 || dims[i] > (int64_t)UINT32_MAX) return dfa_io_fail("tensor dim %lld not representable",
                                                                         (long long)dims[i]);
    if (dims[i] != 0 && n > (int64_t)(SIZE_MAX / 8) / dims[i]) return dfa_io_fail("tensor element count overflows");
    n *= dims[i];
  }
  if (n && !data) return dfa_io_fail("dfa_tensor_save: null data");
  File fh;
  fh.f = fopen(path, "wb");
  if (!fh.f) return dfa_io_fail("cannot open for write: %s", path);
  const uint8_t code = (uint8_t)dtype, rk = (uint8_t)rank;
  bool ok = fwrite(kMagic, 1, 6, fh.f) == 6 && fwrite(&code, 1, 1, fh.f) == 1 && fwrite(&rk, 1, 1, fh.f) == 1;
  for (int i = 0; ok && i < rank; ++i) {
    uint32_t d = (uint32_t)dims[i];
    if (!little_endian()) swap_bytes(&d, 4, 1);
    ok = fwrite(&d, 4, 1, fh.f) == 1;
  }
  const size_t width = dtype == 0 ? 4 : 8;
  if (ok && n) {
    if (little_endian()) {
      ok = fwrite(data, width, (size_t)n, fh.f) == (size_t)n;
    } else {
      std::vector<uint8_t> tmp((const uint8_t*)data, (const uint8_t*)data + (size_t)n * width);
      swap_bytes(tmp.data(), width, (size_t)n);
      ok = fwrite(tmp.data(), width, (size_t)n, fh.f) == (size_t)n;
    }
  }
  if (!ok) return dfa_io_fail("tensor write failed");
  return DFA_OK;
}

}  // extern "C"
