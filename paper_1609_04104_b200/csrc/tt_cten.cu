// CTEN container I/O (reference cten.py:1-74), host side, native.
//
// Layout (little-endian): "CTEN" | u8 version (1) | u8 dtype (0: f32 pairs,
// 1: f64 pairs) | u8 ndim | ndim x u32 dims | payload row-major (re, im).
// The loaders validate exactly what the reference's read_cten rejects
// (magic, version, dtype code, truncated dim table, payload size) and report
// TT_EINVAL with the reference's message shape; Python maps that to
// CtenFormatError(ValueError). tt_cten_read converts straight into a caller
// buffer, complex64 (e.g. pinned memory feeding the device engines) or
// complex128, with several host threads for large payloads.

#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <thread>
#include <vector>

#include "tt_common.cuh"

namespace {

struct CtenHeader {
  int version, dtype, ndim;
  uint32_t dims[32];
  size_t count, offset;  // complex elements, payload byte offset
};

int cten_parse(const char* path, FILE* fh, long fsize, CtenHeader* h) {
  unsigned char head[7];
  if (fsize < 7 || fread(head, 1, 7, fh) != 7 || memcmp(head, "CTEN", 4) != 0)
    return tt_fail(TT_EINVAL, "%s: not a CTEN file", path);
  h->version = head[4];
  h->dtype = head[5];
  h->ndim = head[6];
  if (h->version != 1) return tt_fail(TT_EINVAL, "%s: unsupported CTEN version %d", path, h->version);
  if (h->dtype != 0 && h->dtype != 1) return tt_fail(TT_EINVAL, "%s: unknown dtype code %d", path, h->dtype);
  if (h->ndim > 32) return tt_fail(TT_EUNSUPPORTED, "%s: %d dimensions (at most 32 supported)", path, h->ndim);
  const long hend = 7 + 4L * h->ndim;
  if (fsize < hend) return tt_fail(TT_EINVAL, "%s: truncated dim table", path);
  unsigned char d[4 * 32];
  if (h->ndim && fread(d, 4, (size_t)h->ndim, fh) != (size_t)h->ndim) return tt_fail(TT_EINVAL, "%s: truncated dim table", path);
  size_t count = 1;
  for (int i = 0; i < h->ndim; ++i) {
    h->dims[i] = (uint32_t)d[4 * i] | ((uint32_t)d[4 * i + 1] << 8) | ((uint32_t)d[4 * i + 2] << 16) |
                 ((uint32_t)d[4 * i + 3] << 24);
    count *= h->dims[i];
  }
  h->count = count;
  h->offset = (size_t)hend;
  const size_t esz = h->dtype == 0 ? 8 : 16;
  const size_t expected = (size_t)hend + count * esz;
  if ((size_t)fsize != expected)
    return tt_fail(TT_EINVAL, "%s: payload is %ld bytes, expected %zu", path, fsize - hend, expected - (size_t)hend);
  return TT_OK;
}

int cten_open(const char* path, FILE** fh, long* fsize) {
  *fh = fopen(path, "rb");
  if (!*fh) return tt_fail(TT_EINVAL, "%s: cannot open", path);
  fseek(*fh, 0, SEEK_END);
  *fsize = ftell(*fh);
  fseek(*fh, 0, SEEK_SET);
  return TT_OK;
}

}  // namespace

extern "C" int tt_cten_info(const char* path, int* dtype_code, int* ndim, uint32_t* dims, int max_dims) {
  if (!path || !dtype_code || !ndim) return tt_fail(TT_EINVAL, "tt_cten_info: null argument");
  FILE* fh;
  long fsize;
  int rc = cten_open(path, &fh, &fsize);
  if (rc) return rc;
  CtenHeader h;
  rc = cten_parse(path, fh, fsize, &h);
  fclose(fh);
  if (rc) return rc;
  *dtype_code = h.dtype;
  *ndim = h.ndim;
  if (dims) {
    if (h.ndim > max_dims) return tt_fail(TT_EINVAL, "tt_cten_info: dims buffer too small (%d < %d)", max_dims, h.ndim);
    for (int i = 0; i < h.ndim; ++i) dims[i] = h.dims[i];
  }
  return TT_OK;
}

extern "C" int tt_cten_read(const char* path, void* out, size_t count, int out_is_f64) {
  if (!path || (!out && count)) return tt_fail(TT_EINVAL, "tt_cten_read: null argument");
  FILE* fh;
  long fsize;
  int rc = cten_open(path, &fh, &fsize);
  if (rc) return rc;
  CtenHeader h;
  rc = cten_parse(path, fh, fsize, &h);
  if (rc) {
    fclose(fh);
    return rc;
  }
  if (h.count != count) {
    fclose(fh);
    return tt_fail(TT_EINVAL, "%s: holds %zu elements, buffer has %zu", path, h.count, count);
  }
  const bool same = (h.dtype == 1) == (out_is_f64 != 0);
  if (same) {  // straight into the buffer
    const size_t got = fread(out, h.dtype ? 16 : 8, count, fh);
    fclose(fh);
    if (got != count) return tt_fail(TT_EINVAL, "%s: short read", path);
    return TT_OK;
  }
  const size_t n = 2 * count;
  std::vector<unsigned char> buf(n * (h.dtype ? 8 : 4));
  const size_t got = fread(buf.data(), h.dtype ? 16 : 8, count, fh);
  fclose(fh);
  if (got != count) return tt_fail(TT_EINVAL, "%s: short read", path);
  unsigned nt = std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > 16) nt = 16;
  if (n < (size_t)1 << 20) nt = 1;
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      const size_t a = n * t / nt, b = n * (t + 1) / nt;
      if (h.dtype == 1) {  // f64 pairs -> complex64
        const double* s = (const double*)buf.data();
        float* d = (float*)out;
        for (size_t i = a; i < b; ++i) d[i] = (float)s[i];
      } else {  // f32 pairs -> complex128
        const float* s = (const float*)buf.data();
        double* d = (double*)out;
        for (size_t i = a; i < b; ++i) d[i] = (double)s[i];
      }
    });
  for (auto& th : pool) th.join();
  return TT_OK;
}

extern "C" int tt_cten_write(const char* path, const void* data, int src_is_f64, int dtype_code, int ndim,
                             const uint32_t* dims) {
  if (!path || ndim < 0 || ndim > 32 || (ndim && !dims)) return tt_fail(TT_EINVAL, "tt_cten_write: bad arguments");
  if (dtype_code != 0 && dtype_code != 1) return tt_fail(TT_EINVAL, "unknown dtype code %d", dtype_code);
  size_t count = 1;
  for (int i = 0; i < ndim; ++i) count *= dims[i];
  if (count && !data) return tt_fail(TT_EINVAL, "tt_cten_write: null data");
  FILE* fh = fopen(path, "wb");
  if (!fh) return tt_fail(TT_EINVAL, "%s: cannot open for writing", path);
  unsigned char head[7] = {'C', 'T', 'E', 'N', 1, (unsigned char)dtype_code, (unsigned char)ndim};
  bool ok = fwrite(head, 1, 7, fh) == 7;
  for (int i = 0; ok && i < ndim; ++i) {
    const unsigned char d[4] = {(unsigned char)(dims[i] & 255), (unsigned char)((dims[i] >> 8) & 255),
                                (unsigned char)((dims[i] >> 16) & 255), (unsigned char)(dims[i] >> 24)};
    ok = fwrite(d, 1, 4, fh) == 4;
  }
  const size_t n = 2 * count;
  if (ok && count) {
    const bool same = (dtype_code == 1) == (src_is_f64 != 0);
    if (same) {
      ok = fwrite(data, dtype_code ? 8 : 4, n, fh) == n;
    } else if (dtype_code == 0) {  // f64 source -> f32 pairs
      std::vector<float> buf(n);
      const double* s = (const double*)data;
      for (size_t i = 0; i < n; ++i) buf[i] = (float)s[i];
      ok = fwrite(buf.data(), 4, n, fh) == n;
    } else {  // f32 source -> f64 pairs
      std::vector<double> buf(n);
      const float* s = (const float*)data;
      for (size_t i = 0; i < n; ++i) buf[i] = (double)s[i];
      ok = fwrite(buf.data(), 8, n, fh) == n;
    }
  }
  ok = (fclose(fh) == 0) && ok;
  if (!ok) return tt_fail(TT_EINVAL, "%s: write failed", path);
  return TT_OK;
}
