// Workload-file replay: the reference's binary workload stream
// (include/freescale/workload.hpp:111-144, src/workload.cpp:391-418, 478-549)
// turned into the engine's device input — per-sample UIH lengths, the
// batch-major u64 offsets, the UIH ids and the labels — without building
// per-sample host objects.
//
// Split of work:
//   host  fsx_workload_scan   walks the length prefixes of one iteration
//                             (u32 count per rank, u32 length per record) —
//                             4 bytes per record touched, O(samples); it is
//                             the only inherently sequential part (each record
//                             length locates the next) and it raises the
//                             reference's truncation IoError text.
//   GPU   fsx_workload_decode one thread per record parses the record body
//                             (uih count, candidate lists, label) and checks
//                             it is consumed exactly (the reference's trailing
//                             bytes IoError); u64 offsets scan; the UIH ids
//                             (4-byte aligned in the file, 8-byte aligned in
//                             HBM) move flattened over the output, 2,048 per
//                             CTA tile, coalesced on both sides.
//
// Bytes per record moved on the device: the record once in (H2D of the raw
// iteration), read once by the id mover, ids written once: ~2 x record bytes.
#include <mutex>
#include <string>
#include <unordered_map>

#include "capi_util.cuh"
#include "common.cuh"
#include "table.cuh"

namespace fsx {

void exclusive_offsets(Ctx* ctx, const uint64_t* len, uint64_t n, uint64_t* offs, DevBuf<uint64_t>& scratch,
                       cudaStream_t s);

namespace {

constexpr int kErrRecTruncated = 101;  // a = record, b = iteration-local index
constexpr int kErrRecTrailing = 102;   // a = record
constexpr int kErrIdCapacity = 103;    // a = ids, b = capacity

__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {  // little-endian, 4-byte aligned
  return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ uint64_t ld_u64_a4(const uint8_t* p) {
  return static_cast<uint64_t>(ld_u32(p)) | (static_cast<uint64_t>(ld_u32(p + 4)) << 32);
}

// decode_sample (workload.cpp:405-418) without materialising the candidates:
// uih length + label out, exact-consumption check
__global__ void k_rec_parse(const uint8_t* __restrict__ bytes, uint64_t nbytes, const uint64_t* __restrict__ rec_off,
                            uint64_t n, uint64_t* __restrict__ uih_len, double* __restrict__ labels,
                            DevErr* err) { FSX_PDL_ENTER();
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t off = rec_off[s];
    const uint64_t end = off + ld_u32(bytes + off - 4);  // scan checked end <= nbytes
    uint64_t pos = off;
    bool ok = pos + 4 <= end;
    uint64_t nu = 0;
    if (ok) {
      nu = ld_u32(bytes + pos);
      pos += 4 + 8 * nu;
      ok = pos + 4 <= end;
    }
    if (ok) {
      const uint32_t nc = ld_u32(bytes + pos);
      pos += 4;
      for (uint32_t c = 0; c < nc && ok; ++c) {
        ok = pos + 4 <= end;
        if (ok) pos += 4 + 8 * static_cast<uint64_t>(ld_u32(bytes + pos));
      }
      ok = ok && pos + 8 <= end;
    }
    if (!ok) {
      report(err, kErrRecTruncated, s, 0);
      uih_len[s] = 0;
      continue;
    }
    pos += 8;
    if (pos != end) {
      report(err, kErrRecTrailing, s, 0);
      uih_len[s] = 0;
      continue;
    }
    uih_len[s] = nu;
    if (labels) labels[s] = __longlong_as_double(static_cast<long long>(ld_u64_a4(bytes + pos - 8)));
  }
}

// UIH id mover, flattened over the output ids so a 8,192-id record does not
// serialise one warp (the power-law tail): a CTA takes 2,048 consecutive
// output ids, takes the records that cover them from the tile-first table,
// paints each id's record index into shared memory (warp per record) and then
// moves its ids with 8 loads in flight per thread. Reads (4-byte
// aligned u64 pairs in the file) and writes are coalesced over the tile.
constexpr int kIdTile = 2048;
constexpr int kIdThreads = 256;

__device__ __forceinline__ uint64_t record_of(const uint64_t* offs, uint64_t lo, uint64_t hi, uint64_t x) {
  // last r in [lo, hi) with offs[r] <= x (offs nondecreasing, offs[lo] <= x)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (offs[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// tile_first[t] = the record holding output id t * kIdTile (each tile boundary
// lies in exactly one non-empty record: thread per record, no search);
// tile_first[tiles] = n - 1 closes the last tile's record range
__global__ void k_tile_first(const uint64_t* __restrict__ offs, uint64_t n, uint64_t* __restrict__ tile_first) {
  FSX_PDL_ENTER();
  const uint64_t total = offs[n];
  for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t lo = offs[r], hi = offs[r + 1];
    for (uint64_t t = (lo + kIdTile - 1) / kIdTile; t * kIdTile < hi; ++t) tile_first[t] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) tile_first[(total + kIdTile - 1) / kIdTile] = n - 1;
}

__global__ void __launch_bounds__(kIdThreads) k_rec_ids(const uint8_t* __restrict__ bytes,
                                                        const uint64_t* __restrict__ rec_off, uint64_t n,
                                                        const uint64_t* __restrict__ offs,
                                                        const uint64_t* __restrict__ tile_first,
                                                        uint64_t* __restrict__ values, uint64_t cap, DevErr* err) {
  FSX_PDL_ENTER();
  __shared__ uint16_t sh_rec[kIdTile];
  __shared__ uint64_t sh_base[kIdTile];
  const uint64_t total = offs[n];
  if (total > cap) {  // never write past the caller's buffer
    if (blockIdx.x == 0 && threadIdx.x == 0) report(err, kErrIdCapacity, total, cap);
    return;
  }
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * kIdTile; b < total;
       b += static_cast<uint64_t>(gridDim.x) * kIdTile) {
    const uint64_t e = min(total, b + kIdTile);
    // records [tile_first[t], tile_first[t + 1]] cover the tile (a superset when
    // the next tile's first record starts exactly at e: searches never pick it)
    const uint64_t t = b / kIdTile;
    const uint64_t r0 = tile_first[t], cnt = tile_first[t + 1] - r0 + 1;
    if (cnt <= kIdTile) {
      // paint: sh_rec[id - b] = the id's record (warp per record, lanes over its
      // ids inside the tile); sh_base[k] turns an id into its byte address
      const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
      for (uint64_t k = warp; k < cnt; k += kIdThreads / 32) {
        const uint64_t lo = offs[r0 + k], hi = offs[r0 + k + 1];
        if (lane == 0) sh_base[k] = rec_off[r0 + k] + 4 - 8 * lo;  // mod 2^64
        const uint64_t x1 = min(hi, e);
        for (uint64_t x = max(lo, b) + lane; x < x1; x += 32) sh_rec[x - b] = static_cast<uint16_t>(k);
      }
      __syncthreads();
      constexpr int kPer = kIdTile / kIdThreads;
      const uint8_t* src[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint64_t i = b + threadIdx.x + static_cast<uint64_t>(j) * kIdThreads;
        src[j] = i < e ? bytes + sh_base[sh_rec[i - b]] + 8 * i : nullptr;
      }
      uint64_t v[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j)
        if (src[j]) v[j] = ld_u64_a4(src[j]);
#pragma unroll
      for (int j = 0; j < kPer; ++j)
        if (src[j]) values[b + threadIdx.x + static_cast<uint64_t>(j) * kIdThreads] = v[j];
    } else {  // more than kIdTile records (empty ones) behind 2,048 ids: search in global memory
      for (uint64_t i = b + threadIdx.x; i < e; i += kIdThreads) {
        const uint64_t r = record_of(offs, r0, r0 + cnt, i);
        values[i] = ld_u64_a4(bytes + rec_off[r] + 4 + 8 * (i - offs[r]));
      }
    }
    __syncthreads();
  }
}

// offsets-scan scratch per (context, device), kept across iterations (a
// cudaMalloc / cudaFree pair per call would serialise the device)
DevBuf<uint64_t>& scan_scratch(const Ctx* ctx, int which) {
  static std::mutex m;
  static std::unordered_map<uint64_t, DevBuf<uint64_t>>* bufs = new std::unordered_map<uint64_t, DevBuf<uint64_t>>();
  std::lock_guard<std::mutex> g(m);
  return (*bufs)[(reinterpret_cast<uintptr_t>(ctx) ^ (static_cast<uint64_t>(ctx->device) << 56)) * 2 + which];
}

uint32_t host_u32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

// the reference's Reader::next_iteration truncation text (workload.cpp:511-516)
[[noreturn]] void truncated(int iteration, int rank, long long sample_idx) {
  raise(FSX_ERR_IO, "workload: file truncated; last complete record is iteration " + std::to_string(iteration) +
                        ", rank " + std::to_string(rank) + ", sample " + std::to_string(sample_idx - 1));
}

}  // namespace
}  // namespace fsx

using namespace fsx;

extern "C" {

int fsx_workload_scan(const uint8_t* h_bytes, uint64_t nbytes, int num_ranks, int iteration,
                      uint64_t* h_rank_samples, uint64_t* h_rec_off, uint64_t cap, uint64_t* h_n_records,
                      uint64_t* h_consumed) {
  FSX_API_BEGIN
  if (num_ranks <= 0) raise(FSX_ERR_INVALID_ARGUMENT, "workload: num_ranks must be positive");
  uint64_t pos = 0, k = 0;
  for (int r = 0; r < num_ranks; ++r) {
    if (pos + 4 > nbytes) truncated(iteration, r, 0);
    const uint32_t count = host_u32(h_bytes + pos);
    pos += 4;
    for (uint32_t i = 0; i < count; ++i) {
      if (pos + 4 > nbytes) truncated(iteration, r, i);
      const uint32_t len = host_u32(h_bytes + pos);
      pos += 4;
      if (pos + len > nbytes) truncated(iteration, r, i);
      if (h_rec_off && k < cap) h_rec_off[k] = pos;
      ++k;
      pos += len;
    }
    if (h_rank_samples) h_rank_samples[r] = count;
  }
  if (h_rec_off && k > cap)
    raise(FSX_ERR_INVALID_ARGUMENT,
          "workload: record capacity " + std::to_string(cap) + " below " + std::to_string(k) + " records");
  if (h_n_records) *h_n_records = k;
  if (h_consumed) *h_consumed = pos;
  FSX_API_END
}

int fsx_workload_decode(fsx_ctx* ctx, const uint8_t* d_bytes, uint64_t nbytes, const uint64_t* d_rec_off,
                        uint64_t n, int iteration, const uint64_t* h_rank_samples, int num_ranks,
                        uint64_t* d_uih_len, uint64_t* d_offsets, double* d_labels, uint64_t* d_values,
                        uint64_t cap, uint64_t* h_total, void* stream) {
  FSX_API_BEGIN
  DeviceGuard dg(ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n)
    FSX_LAUNCH(ctx, k_rec_parse, grid_for(ctx, n, 256, 8), 256, 0, s, d_bytes, nbytes, d_rec_off, n, d_uih_len,
               d_labels, ctx->d_err);
  exclusive_offsets(ctx, d_uih_len, n, d_offsets, scan_scratch(ctx, 0), s);
  if (d_values && n) {
    DevBuf<uint64_t>& tf = scan_scratch(ctx, 1);
    tf.ensure(nbytes / 8 / kIdTile + 2);  // ids <= nbytes / 8
    FSX_LAUNCH(ctx, k_tile_first, grid_for(ctx, n, 256, 8), 256, 0, s, d_offsets, n, tf.p);
    FSX_LAUNCH(ctx, k_rec_ids, static_cast<unsigned>(ctx->num_sms) * 8, kIdThreads, 0, s, d_bytes, d_rec_off, n,
               d_offsets, tf.p, d_values, cap, ctx->d_err);
  }
  // one host sync: the error word and the id total together
  uint64_t tot = 0;
  FSX_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaMemcpyAsync(&tot, d_offsets + n, 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  const int kind = ctx->h_err->kind;
  if (kind == kErrRecTruncated || kind == kErrRecTrailing || kind == kErrIdCapacity) {
    const DevErr e = *ctx->h_err;
    FSX_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(DevErr), s));
    FSX_CUDA(cudaStreamSynchronize(s));
    if (kind == kErrRecTruncated) raise(FSX_ERR_IO, "workload: record truncated");  // get_le, workload.cpp:312
    if (kind == kErrIdCapacity)
      raise(FSX_ERR_INVALID_ARGUMENT, "workload: id capacity " + std::to_string(e.b) + " below the iteration's " +
                                          std::to_string(e.a) + " ids");
    uint64_t idx = e.a;
    int r = 0;
    while (r + 1 < num_ranks && h_rank_samples && idx >= h_rank_samples[r]) idx -= h_rank_samples[r++];
    raise(FSX_ERR_IO, "workload: record has trailing bytes at iteration " + std::to_string(iteration) + ", rank " +
                          std::to_string(r) + ", sample " + std::to_string(idx));  // workload.cpp:533-537
  }
  if (kind != kErrNone) ctx->check_error(s);
  if (h_total) *h_total = tot;
  FSX_API_END
}

}  // extern "C"
