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
//                             bytes IoError) and sums its CTA's lengths; a
//                             warp scans the tile sums; the offsets kernel
//                             also marks which record opens each id tile; the
//                             UIH ids
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

namespace {

constexpr int kErrRecTruncated = 101;  // a = record, b = iteration-local index
constexpr int kErrRecTrailing = 102;   // a = record
constexpr int kErrIdCapacity = 103;    // a = ids, b = capacity

// little-endian u32. Valid records are multiples of 4 bytes long, so every
// field sits 4-byte aligned; a record of another length (always malformed,
// the parse reports it) shifts the records behind it, which are then read
// byte by byte instead of faulting with a misaligned access.
__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 3u) == 0) return *reinterpret_cast<const uint32_t*>(p);
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}
__device__ __forceinline__ uint64_t ld_u64_a4(const uint8_t* p) {
  return static_cast<uint64_t>(ld_u32(p)) | (static_cast<uint64_t>(ld_u32(p + 4)) << 32);
}

// UIH id mover, flattened over the output ids so a 8,192-id record does not
// serialise one warp (the power-law tail): a CTA takes 2,048 consecutive
// output ids, takes the records that cover them from the tile-first table,
// paints each id's record index into shared memory (warp per record) and then
// moves its ids with 8 loads in flight per thread. Reads (4-byte
// aligned u64 pairs in the file) and writes are coalesced over the tile.
constexpr int kIdTile = 2048;
constexpr int kIdThreads = 256;

constexpr int kRecTile = 256;  // records per CTA in the parse / offsets kernels

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v) {
  __shared__ uint64_t ws[kRecTile / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  uint64_t t = 0;
#pragma unroll
  for (int w = 0; w < kRecTile / 32; ++w) t += ws[w];
  return t;
}

// decode_sample (workload.cpp:405-418) without materialising the candidates:
// thread per record, uih length + label out, exact-consumption check; the
// CTA's length sum goes to tile_sums for the offsets scan
__global__ void __launch_bounds__(kRecTile) k_rec_parse(const uint8_t* __restrict__ bytes,
                                                        const uint64_t* __restrict__ rec_off, uint64_t n,
                                                        uint64_t* __restrict__ uih_len, double* __restrict__ labels,
                                                        uint64_t* __restrict__ tile_sums,
                                                        unsigned long long* __restrict__ first_bad) {
  FSX_PDL_ENTER();
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * kRecTile + threadIdx.x;
  uint64_t nu = 0;
  if (s < n) {
    const uint64_t off = rec_off[s];
    const uint64_t end = off + ld_u32(bytes + off - 4);  // scan checked end <= nbytes
    uint64_t pos = off;
    bool ok = pos + 4 <= end;
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
    // the reference decodes records in file order and raises at the first
    // bad one: keep the smallest failing record (bit 0: trailing bytes)
    if (!ok) {
      atomicMin(first_bad, static_cast<unsigned long long>(s) << 1);
      nu = 0;
    } else if (pos + 8 != end) {
      atomicMin(first_bad, (static_cast<unsigned long long>(s) << 1) | 1ull);
      nu = 0;
    } else if (labels) {
      labels[s] = __longlong_as_double(static_cast<long long>(ld_u64_a4(bytes + pos)));
    }
    uih_len[s] = nu;
  }
  const uint64_t t = block_sum_u64(nu);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = t;
}

// one warp: exclusive scan of the tile sums in place; offs[n] = total and the
// closing tile_first entry (tile_first[ceil(total / kIdTile)] = n - 1)
__global__ void k_rec_scan_tiles(uint64_t* tile_sums, uint64_t tiles, uint64_t n, uint64_t* __restrict__ offs,
                                 uint64_t* __restrict__ tile_first) {
  FSX_PDL_ENTER();
  const unsigned lane = threadIdx.x & 31u;
  uint64_t carry = 0;
  for (uint64_t t0 = 0; t0 < tiles; t0 += 32) {
    const uint64_t t = t0 + lane;
    const uint64_t v = t < tiles ? tile_sums[t] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (t < tiles) tile_sums[t] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) {
    offs[n] = carry;
    if (tile_first) tile_first[(carry + kIdTile - 1) / kIdTile] = n - 1;
  }
}

// offsets = tile prefix + block exclusive scan of the lengths; each record also
// writes tile_first[t] for every id-tile boundary t * kIdTile it holds
__global__ void __launch_bounds__(kRecTile) k_rec_offsets(const uint64_t* __restrict__ uih_len, uint64_t n,
                                                          const uint64_t* __restrict__ tile_sums,
                                                          uint64_t* __restrict__ offs,
                                                          uint64_t* __restrict__ tile_first) {
  FSX_PDL_ENTER();
  __shared__ uint64_t ws[kRecTile / 32];
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * kRecTile + threadIdx.x;
  const uint64_t v = s < n ? uih_len[s] : 0;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<unsigned>(o)) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  uint64_t lo = tile_sums[blockIdx.x] + x - v;
  for (unsigned w = 0; w < warp; ++w) lo += ws[w];
  if (s < n) {
    offs[s] = lo;
    if (tile_first)
      for (uint64_t t = (lo + kIdTile - 1) / kIdTile; t * kIdTile < lo + v; ++t) tile_first[t] = s;
  }
}


__device__ __forceinline__ uint64_t record_of(const uint64_t* offs, uint64_t lo, uint64_t hi, uint64_t x) {
  // last r in [lo, hi) with offs[r] <= x (offs nondecreasing, offs[lo] <= x)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (offs[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
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

// decode_sample's structure check of one record on the host (workload.cpp:
// 405-418): 0 = decodes exactly, 1 = truncated, 2 = trailing bytes. Only the
// error path uses it (see truncated_after).
int host_record_status(const uint8_t* rec, uint64_t len) {
  uint64_t pos = 0;
  if (pos + 4 > len) return 1;
  const uint64_t nu = host_u32(rec + pos);
  pos += 4 + 8 * nu;
  if (pos + 4 > len) return 1;
  const uint32_t nc = host_u32(rec + pos);
  pos += 4;
  for (uint32_t c = 0; c < nc; ++c) {
    if (pos + 4 > len) return 1;
    pos += 4 + 8 * static_cast<uint64_t>(host_u32(rec + pos));
  }
  if (pos + 8 > len) return 1;
  return pos + 8 == len ? 0 : 2;
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
  // The reference decodes each record as it reads it (workload.cpp:518-537),
  // so a malformed record before the truncation point raises first: on
  // truncation, re-walk the complete records in file order and raise the
  // first one's decode error, else the truncation.
  auto truncated_after = [&](int rr, long long ii) {
    uint64_t q = 0;
    for (int r2 = 0; r2 <= rr; ++r2) {
      const uint32_t cnt = host_u32(h_bytes + q);
      q += 4;
      for (uint32_t i2 = 0; i2 < cnt && (r2 < rr || i2 < static_cast<uint64_t>(ii)); ++i2) {
        const uint32_t len2 = host_u32(h_bytes + q);
        q += 4;
        const int st = host_record_status(h_bytes + q, len2);
        if (st == 1) raise(FSX_ERR_IO, "workload: record truncated");
        if (st == 2)
          raise(FSX_ERR_IO, "workload: record has trailing bytes at iteration " + std::to_string(iteration) +
                                ", rank " + std::to_string(r2) + ", sample " + std::to_string(i2));
        q += len2;
      }
    }
    truncated(iteration, rr, ii);
  };
  for (int r = 0; r < num_ranks; ++r) {
    if (pos + 4 > nbytes) truncated_after(r, 0);
    const uint32_t count = host_u32(h_bytes + pos);
    pos += 4;
    for (uint32_t i = 0; i < count; ++i) {
      if (pos + 4 > nbytes) truncated_after(r, i);
      const uint32_t len = host_u32(h_bytes + pos);
      pos += 4;
      if (pos + len > nbytes) truncated_after(r, i);
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
  uint64_t* first_bad = nullptr;
  if (n) {
    const uint64_t tiles = (n + kRecTile - 1) / kRecTile;
    DevBuf<uint64_t>& ts = scan_scratch(ctx, 0);
    ts.ensure(tiles);
    uint64_t* tf = nullptr;
    if (d_values) {
      DevBuf<uint64_t>& tfb = scan_scratch(ctx, 1);
      tfb.ensure(nbytes / 8 / kIdTile + 2);  // ids <= nbytes / 8
      tf = tfb.p;
    }
    DevBuf<uint64_t>& fb = scan_scratch(ctx, 2);
    fb.ensure(1);
    first_bad = fb.p;
    FSX_CUDA(cudaMemsetAsync(first_bad, 0xff, 8, s));
    FSX_LAUNCH(ctx, k_rec_parse, static_cast<unsigned>(tiles), kRecTile, 0, s, d_bytes, d_rec_off, n, d_uih_len,
               d_labels, ts.p, reinterpret_cast<unsigned long long*>(first_bad));
    FSX_LAUNCH(ctx, k_rec_scan_tiles, 1, 32, 0, s, ts.p, tiles, n, d_offsets, tf);
    FSX_LAUNCH(ctx, k_rec_offsets, static_cast<unsigned>(tiles), kRecTile, 0, s, d_uih_len, n, ts.p, d_offsets, tf);
    if (d_values)
      FSX_LAUNCH(ctx, k_rec_ids, static_cast<unsigned>(ctx->num_sms) * 8, kIdThreads, 0, s, d_bytes, d_rec_off, n,
                 d_offsets, tf, d_values, cap, ctx->d_err);
  } else {
    FSX_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(uint64_t), s));
  }
  // one host sync: the error word and the id total together
  uint64_t tot = 0, bad = ~0ull;
  FSX_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaMemcpyAsync(&tot, d_offsets + n, 8, cudaMemcpyDeviceToHost, s));
  if (first_bad) FSX_CUDA(cudaMemcpyAsync(&bad, first_bad, 8, cudaMemcpyDeviceToHost, s));
  FSX_CUDA(cudaStreamSynchronize(s));
  const int kind = bad != ~0ull ? ((bad & 1u) ? kErrRecTrailing : kErrRecTruncated) : ctx->h_err->kind;
  if (kind == kErrRecTruncated || kind == kErrRecTrailing || kind == kErrIdCapacity) {
    const DevErr e = bad != ~0ull ? DevErr{kind, 0, bad >> 1, 0} : *ctx->h_err;
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
