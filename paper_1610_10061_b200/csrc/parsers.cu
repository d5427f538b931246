// Instance ingestion: the reference's text formats.
//
//  * OR-Library graph format -- pmedian::parse_orlib (proj/src/bench.cpp:106-168):
//    token stream "n edges p" then "u v cost" triples (1-based), parallel
//    edges keep the cheapest, the instance is the all-pairs shortest-path
//    closure, a disconnected graph is rejected.  Tokenising and validation run
//    on the host with the reference's diagnostics; the closure runs on the
//    device as a blocked Floyd-Warshall (32x32 int64 min-plus tiles) and lands
//    directly in the device cost matrix K1 sorts, so pmed-sized instances never
//    round-trip through host memory.  The min-plus closure is unique, so the
//    result is the reference's matrix exactly, sentinel included
//    (kUnreachable = INT64_MAX / 4, bench.cpp:123).
//  * dense format -- pmedian::parse_dense (bench.cpp:65-104): host parsing.
#include <cuda_runtime.h>

#include <cctype>
#include <charconv>
#include <algorithm>
#include <climits>
#include <string>
#include <string_view>
#include <vector>

#include "common.cuh"
#include "ctx.h"

namespace pmb {

constexpr int64_t kUnreachable = INT64_MAX / 4;  // bench.cpp:123
constexpr int kFwTile = 32;

// ---- device Floyd-Warshall ----------------------------------------------------------

__global__ void k_fw_init(int64_t* __restrict__ d, int nP, int n) {
  const size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (x >= (size_t)nP * nP) return;
  const int i = (int)(x / nP), j = (int)(x % nP);
  d[x] = (i == j && i < n) ? 0 : kUnreachable;
}

// parallel edges keep the cheapest (bench.cpp:141-143)
__global__ void k_fw_edges(int64_t* __restrict__ d, int nP, const int* __restrict__ uv,
                           const int64_t* __restrict__ w, int edges) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= edges) return;
  const int a = uv[2 * e], b = uv[2 * e + 1];
  atomicMin(reinterpret_cast<long long*>(d + (size_t)a * nP + b), (long long)w[e]);
  atomicMin(reinterpret_cast<long long*>(d + (size_t)b * nP + a), (long long)w[e]);
}

__device__ __forceinline__ int64_t relax(int64_t cur, int64_t a, int64_t b) {
  const int64_t t = a + b;  // both <= kUnreachable: no overflow
  return t < cur ? t : cur;
}

// phase 1: the pivot tile against itself
__global__ void k_fw_pivot(int64_t* __restrict__ d, int nP, int kb) {
  __shared__ int64_t s[kFwTile][kFwTile + 1];
  const int ty = threadIdx.y, tx = threadIdx.x, o = kb * kFwTile;
  s[ty][tx] = d[(size_t)(o + ty) * nP + o + tx];
  __syncthreads();
  for (int k = 0; k < kFwTile; ++k) {
    const int64_t v = relax(s[ty][tx], s[ty][k], s[k][tx]);
    __syncthreads();
    s[ty][tx] = v;
    __syncthreads();
  }
  d[(size_t)(o + ty) * nP + o + tx] = s[ty][tx];
}

// phase 2: tiles of the pivot row (blockIdx.y == 0) and pivot column (== 1)
__global__ void k_fw_cross(int64_t* __restrict__ d, int nP, int kb) {
  const int t = blockIdx.x >= (unsigned)kb ? blockIdx.x + 1 : blockIdx.x;  // skip the pivot
  __shared__ int64_t p[kFwTile][kFwTile + 1], s[kFwTile][kFwTile + 1];
  const int ty = threadIdx.y, tx = threadIdx.x, o = kb * kFwTile;
  const bool row = blockIdx.y == 0;
  const int r0 = row ? o : t * kFwTile, c0 = row ? t * kFwTile : o;
  p[ty][tx] = d[(size_t)(o + ty) * nP + o + tx];
  s[ty][tx] = d[(size_t)(r0 + ty) * nP + c0 + tx];
  __syncthreads();
  for (int k = 0; k < kFwTile; ++k) {
    const int64_t v = row ? relax(s[ty][tx], p[ty][k], s[k][tx]) : relax(s[ty][tx], s[ty][k], p[k][tx]);
    __syncthreads();
    s[ty][tx] = v;
    __syncthreads();
  }
  d[(size_t)(r0 + ty) * nP + c0 + tx] = s[ty][tx];
}

// phase 3: every other tile, a min-plus product of its row and column tiles
__global__ void k_fw_rest(int64_t* __restrict__ d, int nP, int kb) {
  const int bi = blockIdx.y >= (unsigned)kb ? blockIdx.y + 1 : blockIdx.y;
  const int bj = blockIdx.x >= (unsigned)kb ? blockIdx.x + 1 : blockIdx.x;
  __shared__ int64_t a[kFwTile][kFwTile + 1], b[kFwTile][kFwTile + 1];
  const int ty = threadIdx.y, tx = threadIdx.x, o = kb * kFwTile;
  a[ty][tx] = d[(size_t)(bi * kFwTile + ty) * nP + o + tx];
  b[ty][tx] = d[(size_t)(o + ty) * nP + bj * kFwTile + tx];
  __syncthreads();
  int64_t v = d[(size_t)(bi * kFwTile + ty) * nP + bj * kFwTile + tx];
#pragma unroll 8
  for (int k = 0; k < kFwTile; ++k) v = relax(v, a[ty][k], b[k][tx]);
  d[(size_t)(bi * kFwTile + ty) * nP + bj * kFwTile + tx] = v;
}

// compact to n x n and find the first unreachable pair in row-major order
__global__ void k_fw_finish(const int64_t* __restrict__ d, int nP, int n, int64_t* __restrict__ out,
                            unsigned long long* __restrict__ first_bad) {
  const size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (x >= (size_t)n * n) return;
  const int i = (int)(x / n), j = (int)(x % n);
  const int64_t v = d[(size_t)i * nP + j];
  out[x] = v;
  if (v >= kUnreachable) atomicMin(first_bad, (unsigned long long)x);
}

// ---- host tokenising (bench.cpp:21-60) ------------------------------------------------

static std::vector<std::string_view> split_tokens(std::string_view text) {
  std::vector<std::string_view> tokens;
  size_t i = 0;
  while (i < text.size()) {
    while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
    size_t j = i;
    while (j < text.size() && !std::isspace(static_cast<unsigned char>(text[j]))) ++j;
    if (j > i) tokens.push_back(text.substr(i, j - i));
    i = j;
  }
  return tokens;
}

struct ParseError {
  int code;
  std::string msg;
};

static int64_t parse_int(std::string_view tok, const char* what) {
  int64_t v = 0;
  const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || ptr != tok.data() + tok.size())
    throw ParseError{PM_STRUCTURAL, std::string("could not parse ") + what + ": '" + std::string(tok) + "'"};
  return v;
}

// Validates the graph text exactly as parse_orlib does (bench.cpp:108-139) and
// runs the closure on the device; `out` receives the n x n matrix (device).
static int orlib_closure(pm_ctx* c, std::string_view text, DevBuf& out, size_t* n_out, size_t* p_out) {
  std::vector<int> uv;
  std::vector<int64_t> w;
  int64_t n = 0, p = 0;
  try {
    const auto tokens = split_tokens(text);
    if (tokens.size() < 3) throw ParseError{PM_STRUCTURAL, "graph format: header must be 'n edges p'"};
    n = parse_int(tokens[0], "vertex count");
    const int64_t edges = parse_int(tokens[1], "edge count");
    p = parse_int(tokens[2], "p");
    if (n < 1) throw ParseError{PM_STRUCTURAL, "graph format: vertex count must be positive"};
    if (edges < 0) throw ParseError{PM_STRUCTURAL, "graph format: edge count must be non-negative"};
    if (tokens.size() != 3 + 3 * (size_t)edges)
      throw ParseError{PM_STRUCTURAL, "graph format: expected " + std::to_string(edges) +
                                          " 'u v cost' triples, found " + std::to_string((tokens.size() - 3) / 3) +
                                          " plus stray tokens"};
    if (n > 65536) throw ParseError{PM_DOMAIN, "graph format: at most 65536 vertices on the device"};
    uv.reserve(2 * edges);
    w.reserve(edges);
    for (int64_t e = 0; e < edges; ++e) {
      const size_t b = 3 + 3 * (size_t)e;
      const int64_t u = parse_int(tokens[b], "edge endpoint");
      const int64_t v = parse_int(tokens[b + 1], "edge endpoint");
      const int64_t cost = parse_int(tokens[b + 2], "edge cost");
      if (u < 1 || u > n || v < 1 || v > n)
        throw ParseError{PM_STRUCTURAL, "graph format: vertex index out of range in edge " + std::to_string(e + 1)};
      if (cost < 0)
        throw ParseError{PM_STRUCTURAL, "graph format: negative cost on edge " + std::to_string(e + 1)};
      uv.push_back((int)(u - 1));
      uv.push_back((int)(v - 1));
      w.push_back(cost);
    }
  } catch (const ParseError& e) {
    return c->fail(e.code, e.msg);
  }
  const int N = (int)n, nP = (N + kFwTile - 1) / kFwTile * kFwTile, nb = nP / kFwTile;
  DevBuf mat, duv, dw, bad;
  PM_CUDA_TRY(c, mat.ensure((size_t)nP * nP * 8));
  PM_CUDA_TRY(c, out.ensure((size_t)N * N * 8));
  PM_CUDA_TRY(c, bad.ensure(8));
  const int E = (int)w.size();
  cudaStream_t st = c->stream;
  k_fw_init<<<(unsigned)(((size_t)nP * nP + 255) / 256), 256, 0, st>>>(mat.as<int64_t>(), nP, N);
  if (E > 0) {
    PM_CUDA_TRY(c, duv.ensure(uv.size() * 4));
    PM_CUDA_TRY(c, dw.ensure(w.size() * 8));
    PM_CUDA_TRY(c, cudaMemcpyAsync(duv.p, uv.data(), uv.size() * 4, cudaMemcpyHostToDevice, st));
    PM_CUDA_TRY(c, cudaMemcpyAsync(dw.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice, st));
    k_fw_edges<<<(E + 255) / 256, 256, 0, st>>>(mat.as<int64_t>(), nP, duv.as<int>(), dw.as<int64_t>(), E);
  }
  const dim3 tile(kFwTile, kFwTile);
  for (int kb = 0; kb < nb; ++kb) {
    k_fw_pivot<<<1, tile, 0, st>>>(mat.as<int64_t>(), nP, kb);
    if (nb > 1) {
      k_fw_cross<<<dim3(nb - 1, 2), tile, 0, st>>>(mat.as<int64_t>(), nP, kb);
      k_fw_rest<<<dim3(nb - 1, nb - 1), tile, 0, st>>>(mat.as<int64_t>(), nP, kb);
    }
  }
  PM_CUDA_TRY(c, cudaMemsetAsync(bad.p, 0xff, 8, st));
  k_fw_finish<<<(unsigned)(((size_t)N * N + 255) / 256), 256, 0, st>>>(mat.as<int64_t>(), nP, N, out.as<int64_t>(),
                                                                       bad.as<unsigned long long>());
  PM_CUDA_TRY(c, cudaGetLastError());
  c->launches += 3 + 3 * (size_t)nb;
  unsigned long long first = 0;
  PM_CUDA_TRY(c, cudaMemcpyAsync(&first, bad.p, 8, cudaMemcpyDeviceToHost, st));
  PM_CUDA_TRY(c, cudaStreamSynchronize(st));
  for (DevBuf* b : {&mat, &duv, &dw, &bad}) b->release();
  if (first != ~0ull) {  // bench.cpp:159-166
    const size_t i = first / N, j = first % N;
    return c->fail(PM_STRUCTURAL, "graph format: disconnected graph, no path between vertices " +
                                      std::to_string(i + 1) + " and " + std::to_string(j + 1));
  }
  *n_out = (size_t)N;
  *p_out = (size_t)p;
  return PM_OK;
}

}  // namespace pmb

using namespace pmb;

extern "C" {

int pm_orlib_closure(pm_ctx* c, const char* text, size_t len, int64_t* costs_out, size_t capacity,
                     size_t* n_out, size_t* p_out) {
  if (!c) return PM_STRUCTURAL;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  DevBuf out;
  size_t n = 0, p = 0;
  int rc = orlib_closure(c, std::string_view(text ? text : "", text ? len : 0), out, &n, &p);
  if (rc != PM_OK) return rc;
  if (n_out) *n_out = n;
  if (p_out) *p_out = p;
  if (costs_out) {
    if (capacity < n * n) {
      out.release();
      return c->fail(PM_STRUCTURAL, "output buffer smaller than n * n");
    }
    PM_CUDA_TRY(c, cudaMemcpy(costs_out, out.p, n * n * 8, cudaMemcpyDeviceToHost));
  }
  out.release();
  return PM_OK;
}

int pm_set_instance_orlib(pm_ctx* c, const char* text, size_t len, size_t p_override) {
  if (!c) return PM_STRUCTURAL;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  DevBuf out;
  size_t n = 0, p = 0;
  int rc = orlib_closure(c, std::string_view(text ? text : "", text ? len : 0), out, &n, &p);
  if (rc != PM_OK) return rc;
  rc = pm_set_instance_device(c, out.as<int64_t>(), n, n, p_override ? p_override : p);
  out.release();
  return rc;
}

// parse_dense (bench.cpp:65-104) on the host: diagnostics in the reference's order and texts.
static int parse_dense_host(pm_ctx* c, const char* text, size_t len, std::vector<int64_t>& costs, int64_t& n,
                            int64_t& m, int64_t& p) {
  const std::string_view t(text ? text : "", text ? len : 0);
  std::vector<std::string_view> lines;
  size_t start = 0;
  while (start <= t.size()) {
    const size_t end = t.find('\n', start);
    const std::string_view line = t.substr(start, end == std::string_view::npos ? std::string_view::npos : end - start);
    bool blank = true;
    for (char ch : line) blank &= std::isspace(static_cast<unsigned char>(ch)) != 0;
    if (!blank) lines.push_back(line);
    if (end == std::string_view::npos) break;
    start = end + 1;
  }
  try {
    if (lines.empty()) throw ParseError{PM_STRUCTURAL, "dense format: empty input"};
    const auto header = split_tokens(lines[0]);
    if (header.size() != 3) throw ParseError{PM_STRUCTURAL, "dense format: header must be 'n m p'"};
    n = parse_int(header[0], "n");
    m = parse_int(header[1], "m");
    p = parse_int(header[2], "p");
    if (n < 1) throw ParseError{PM_STRUCTURAL, "dense format: n must be positive"};
    if (m < 1) throw ParseError{PM_STRUCTURAL, "dense format: m must be positive"};
    if (p < 1) throw ParseError{PM_DOMAIN, "p must be >= 1"};
    if (lines.size() - 1 != (size_t)n)
      throw ParseError{PM_STRUCTURAL, "dense format: expected " + std::to_string(n) + " cost rows, found " +
                                          std::to_string(lines.size() - 1)};
    costs.clear();
    costs.reserve((size_t)n * m);
    for (int64_t i = 0; i < n; ++i) {
      const auto row = split_tokens(lines[(size_t)i + 1]);
      if (row.size() != (size_t)m)
        throw ParseError{PM_STRUCTURAL, "dense format: row " + std::to_string(i + 1) + " has " +
                                            std::to_string(row.size()) + " values, expected " + std::to_string(m)};
      for (int64_t j = 0; j < m; ++j) {
        const int64_t v = parse_int(row[(size_t)j], "cost");
        if (v < 0)
          throw ParseError{PM_STRUCTURAL, "dense format: negative cost at row " + std::to_string(i + 1) +
                                              ", column " + std::to_string(j + 1)};
        costs.push_back(v);
      }
    }
  } catch (const ParseError& e) {
    return c->fail(e.code, e.msg);
  }
  return PM_OK;
}

int pm_set_instance_dense(pm_ctx* c, const char* text, size_t len, size_t p_override) {
  if (!c) return PM_STRUCTURAL;
  std::vector<int64_t> costs;
  int64_t n = 0, m = 0, p = 0;
  const int rc = parse_dense_host(c, text, len, costs, n, m, p);
  if (rc != PM_OK) return rc;
  return pm_set_instance(c, costs.data(), (size_t)n, (size_t)m, p_override ? p_override : (size_t)p);
}

int pm_parse_dense(pm_ctx* c, const char* text, size_t len, int64_t* costs_out, size_t capacity, size_t* n_out,
                   size_t* m_out, size_t* p_out) {
  if (!c) return PM_STRUCTURAL;
  std::vector<int64_t> costs;
  int64_t n = 0, m = 0, p = 0;
  const int rc = parse_dense_host(c, text, len, costs, n, m, p);
  if (rc != PM_OK) return rc;
  if (n_out) *n_out = (size_t)n;
  if (m_out) *m_out = (size_t)m;
  if (p_out) *p_out = (size_t)p;
  if (costs_out) {
    if (capacity < costs.size()) return c->fail(PM_STRUCTURAL, "output buffer smaller than n * m");
    std::copy(costs.begin(), costs.end(), costs_out);
  }
  return PM_OK;
}

}  // extern "C"
