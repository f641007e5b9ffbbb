// Host-side helpers shared by the HBS translation units (hbs.cu: compress /
// apply / invert / DTNHBS01; hbs_ops.cu: the HBS algebra): descriptor upload,
// batched launches, the pooled scratch and the factor arena.
#pragma once

#include <atomic>
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "hbs.hpp"

namespace dtnb {

template <class T>
inline void pmalloc(T** p, size_t bytes) {
  *p = static_cast<T*>(pool_alloc(bytes));
}

cudaError_t launch_gemm_desc(const GemmDesc* d_descs, int count, int max_tiles, int kmax, double alpha, double beta,
                             cudaStream_t st, bool a_aligned, bool allow_big = true);
cudaError_t launch_gemm_desc_tc(const GemmDesc* d_descs, int count, int max_tiles, int kmax, double alpha, double beta,
                                cudaStream_t st);
cudaError_t launch_gemm_desc2(const GemmDesc2* d_descs, int count, int max_tiles, bool tc, cudaStream_t st);
int gemm_tiles(int m, int n);
cudaError_t launch_hqr(const QrDesc* d_descs, int count, int max_m, int max_nc, const double* d_eps, cudaStream_t st,
                       bool pivoted);
cudaError_t launch_fill_uniform(double* X, int ldx, int rows, int cols, unsigned long long seed, cudaStream_t st);
cudaError_t launch_copy2d_batched(const void* d_descs, int count, cudaStream_t st);
cudaError_t launch_sum_slices(double* base, long long stride, int slices, long long count, cudaStream_t st);

// kernel launches issued by the HBS code (compress, invert, apply), process-wide
extern std::atomic<unsigned long long> g_hbs_launches;

#define HLK(x)                    \
  do {                            \
    HCK(x);                       \
    g_hbs_launches.fetch_add(1);  \
  } while (0)

#define HCK(x)                                                                                        \
  do {                                                                                                \
    const cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                                    " at " #x);                                       \
  } while (0)

namespace {
inline int64_t align2(int64_t x) { return (x + 1) & ~int64_t(1); }

}  // namespace

// Device scratch for descriptors and staging: every get() is a FRESH region (a bump
// allocator over pooled chunks), never reused while the owning call runs, so a launch
// never waits for the previous one to have read its descriptors (no synchronisation
// between batches). The owner synchronises its stream before the chunks return to the
// pool (every user ends with a stream synchronisation).
struct DevBuf {
  std::vector<void*> chunks;
  char* cur = nullptr;
  size_t cap = 0, off = 0;
  ~DevBuf() {
    for (void* c : chunks) pool_free(c);
  }
  void* get(size_t bytes) {
    bytes = (std::max<size_t>(bytes, 1) + 255) & ~size_t(255);
    if (!cur || off + bytes > cap) {
      const size_t c = std::max<size_t>(bytes, size_t(1) << 20);
      void* q = nullptr;
      pmalloc(&q, c);
      chunks.push_back(q);
      cur = static_cast<char*>(q);
      cap = c;
      off = 0;
    }
    void* r = cur + off;
    off += bytes;
    return r;
  }
};

namespace {
// host descriptors -> device, then launch
template <class T>
T* upload(DevBuf& buf, const std::vector<T>& v, cudaStream_t st) {
  T* d = static_cast<T*>(buf.get(v.size() * sizeof(T)));
  if (!v.empty()) HCK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return d;
}

void gemm_batch(DevBuf& buf, const std::vector<GemmDesc>& g, double alpha, double beta, bool a_aligned,
                cudaStream_t st) {
  if (g.empty()) return;
  int tiles = 0, kmax = 0;
  for (const auto& d : g) {
    if (d.m <= 0 || d.n <= 0) continue;
    tiles = std::max(tiles, gemm_tiles(d.m, d.n));
    kmax = std::max(kmax, d.k);
  }
  if (tiles == 0) return;
  GemmDesc* dd = upload(buf, g, st);
  HLK(launch_gemm_desc(dd, int(g.size()), tiles, kmax, alpha, beta, st, a_aligned));
}

void transpose_batch(DevBuf& buf, const std::vector<TransDesc>& t, cudaStream_t st) {
  if (t.empty()) return;
  int tiles = 0;
  for (const auto& d : t) tiles = std::max(tiles, ((d.m + 31) / 32) * ((d.n + 31) / 32));
  TransDesc* dd = upload(buf, t, st);
  HLK(launch_transpose_batched(dd, int(t.size()), tiles, st));
}

void copy_batch(DevBuf& buf, const std::vector<CopyDesc>& c, cudaStream_t st) {
  if (c.empty()) return;
  // large blocks (the M x M working matrix) go through the copy engine; the
  // batched kernel is for many small blocks
  std::vector<CopyDesc> small;
  for (const auto& d : c) {
    if (int64_t(d.m) * d.n >= (int64_t(1) << 20))
      HCK(cudaMemcpy2DAsync(d.dst, size_t(d.ldd) * 8, d.src, size_t(d.lds) * 8, size_t(d.m) * 8, size_t(d.n),
                            cudaMemcpyDeviceToDevice, st));
    else if (d.m > 0 && d.n > 0)
      small.push_back(d);
  }
  if (!small.empty()) {
    CopyDesc* dd = upload(buf, small, st);
    HLK(launch_copy2d_batched(dd, int(small.size()), st));
  }
}

}  // namespace

// Grow-only device scratch of the compression (the M x M work matrices are
// 2 GB each at M = 16380): kept per device between calls instead of
// cudaMalloc/cudaFree per call; one compression at a time per device.
struct Scratch {
  std::mutex m;
  std::vector<std::pair<void*, size_t>> slot;
  void* get(int i, size_t bytes) {
    if (int(slot.size()) <= i) slot.resize(i + 1, {nullptr, 0});
    auto& e = slot[i];
    if (e.second < bytes) {
      if (e.first) pool_free(e.first);
      e = {nullptr, 0};
      pmalloc(&e.first, bytes);
      e.second = bytes;
    }
    return e.first;
  }
};

// Owned factor storage of one HbsDev, handed out from a few large chunks
// (one cudaMalloc per chunk instead of one per tree level and factor kind).
struct Arena {
  HbsDev& H;
  size_t chunk;
  double* cur = nullptr;
  size_t left = 0;
  Arena(HbsDev& h, size_t first_chunk_doubles) : H(h), chunk(std::max<size_t>(first_chunk_doubles, 1 << 16)) {}
  double* alloc(size_t doubles) {
    doubles = (doubles + 1) & ~size_t(1);  // keep 16-byte alignment
    if (doubles > left) {
      const size_t sz = std::max(doubles, chunk);
      void* p = nullptr;
      pmalloc(&p, sz * 8);
      H.buffers.push_back(p);
      cur = static_cast<double*>(p);
      left = sz;
      chunk *= 2;
    }
    double* r = cur;
    cur += doubles;
    left -= doubles;
    return r;
  }
};

// per-device grow-only scratch of the compression (hbs.cu)
Scratch& scratch(int device);

}  // namespace dtnb
