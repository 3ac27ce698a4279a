// Device Gaussian test matrix Omega, bit-identical to the reference's
//   Generator(Philox(SeedSequence([seed, 0x534B, ncols, w]))).standard_normal((ncols, w))
// (matcore.py:89-92, rsvd.py:56).  SURVEY §8(f) rank 1.
//
// NumPy draws each normal from a variable number of Philox4x64-10 words (one on the ~99 %
// ziggurat fast path, more on the slow paths), so the stream is consumed sequentially.  On
// the device:
//   1. every Philox block (4 words) is generated independently from its counter;
//   2. for every word position i, one thread simulates a complete draw that would START at i
//      (value, words consumed) — independent of where draws actually start;
//   3. the chain of actual start positions 0, 0 + c(0), ... is resolved hierarchically:
//      per 256-word segment the (outputs, exit offset) map for each small entry offset, maps
//      composed per 256-segment chunk, one thread over the chunks, then per segment again;
//   4. each segment writes its outputs to their global indices.
// The ziggurat constants are measured from the installed NumPy (tools/probe_ziggurat.py).
// The slow paths' accept tests use the device exp/log1p (a flip against the host libm needs a
// uniform within ~1 ulp of the threshold); the few tail values (~1e-4 of draws) are recomputed
// on the host with the same libm log1p NumPy calls, so every value is bit-identical.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "ziggurat_tables.h"

namespace lramm {
namespace {

constexpr uint64_t kPhM0 = 0xD2E7470EE14C6C93ULL, kPhM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kPhW0 = 0x9E3779B97F4A7C15ULL, kPhW1 = 0xBB67AE8584CAA73BULL;
constexpr int kSeg = 256;    // words per segment
constexpr int kEntries = 4;  // precomputed entry offsets per segment
constexpr int kChunk = 256;  // segments per chunk
constexpr uint8_t kBadConsume = 255;
constexpr int kTailWords = 32;  // words kept per tail draw for the host recomputation

__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kPhW0;
      k1 += kPhW1;
    }
    const uint64_t hi0 = __umul64hi(kPhM0, c[0]), lo0 = kPhM0 * c[0];
    const uint64_t hi1 = __umul64hi(kPhM1, c[2]), lo1 = kPhM1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// word j = output (j % 4) of the block with counter j / 4 + 1 (NumPy increments before use)
__global__ void philox_kernel(uint64_t *__restrict__ raw, int64_t nraw, uint64_t k0, uint64_t k1) {
  const int64_t nblk = (nraw + 3) / 4;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {(uint64_t)b + 1, 0, 0, 0};
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * b + q < nraw) raw[4 * b + q] = c[q];
  }
}

__device__ __forceinline__ double u53(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }

// one complete standard_normal draw starting at word i: value, words consumed, tail flag
__global__ void attempt_kernel(const uint64_t *__restrict__ raw, int64_t nraw, uint8_t *__restrict__ consume,
                               double *__restrict__ value, uint8_t *__restrict__ tail) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nraw; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = i;
    double out = 0.0;
    uint8_t is_tail = 0;
    bool ok = false;
    while (j < nraw && j - i < 200) {
      uint64_t r = raw[j++];
      const int idx = (int)(r & 0xFF);
      r >>= 8;
      const int sign = (int)(r & 1);
      const uint64_t rabs = (r >> 1) & 0x000FFFFFFFFFFFFFULL;
      double x = (double)rabs * kZigW[idx];
      if (sign) x = -x;
      if (rabs < kZigK[idx]) {
        out = x;
        ok = true;
        break;
      }
      if (idx == 0) {
        bool done = false;
        while (j + 1 < nraw && j - i < 200) {
          const double xx = -kZigInvR * log1p(-u53(raw[j]));
          const double yy = -log1p(-u53(raw[j + 1]));
          j += 2;
          if (yy + yy > xx * xx) {
            out = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
            is_tail = 1;
            done = true;
            break;
          }
        }
        if (done) ok = true;
        break;
      }
      if (j >= nraw) break;
      const double u = u53(raw[j++]);
      if ((kZigF[idx - 1] - kZigF[idx]) * u + kZigF[idx] < exp(-0.5 * x * x)) {
        out = x;
        ok = true;
        break;
      }
    }
    consume[i] = ok ? (uint8_t)(j - i) : kBadConsume;
    value[i] = out;
    tail[i] = is_tail;
  }
}

// walk the chain through one segment from entry offset e: outputs started inside the segment
// and the entry offset into the next segment (kBadConsume: ran off the generated words)
__device__ __forceinline__ void seg_walk(const uint8_t *consume, int64_t nraw, int64_t s, int e, int &cnt, int &nxt) {
  int64_t pos = s * kSeg + e;
  const int64_t end = (s + 1) * kSeg;
  cnt = 0;
  while (pos < end) {
    if (pos >= nraw || consume[pos] == kBadConsume) {
      nxt = -1;
      return;
    }
    pos += consume[pos];
    ++cnt;
  }
  nxt = (int)(pos - end);
}

__global__ void seg_map_kernel(const uint8_t *__restrict__ consume, int64_t nraw, int64_t nseg, int *__restrict__ cnt,
                               int *__restrict__ nxt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nseg * kEntries;
       t += (int64_t)gridDim.x * blockDim.x) {
    int c, n;
    seg_walk(consume, nraw, t / kEntries, (int)(t % kEntries), c, n);
    cnt[t] = c;
    nxt[t] = n;
  }
}

__device__ __forceinline__ void seg_step(const uint8_t *consume, int64_t nraw, const int *cnt, const int *nxt,
                                         int64_t s, int e, int &c, int &n) {
  if (e >= 0 && e < kEntries) {
    c = cnt[s * kEntries + e];
    n = nxt[s * kEntries + e];
  } else {
    seg_walk(consume, nraw, s, e, c, n);
  }
}

// chunk maps: for each chunk and entry offset, outputs over the chunk and the exit offset
__global__ void chunk_map_kernel(const uint8_t *__restrict__ consume, int64_t nraw, int64_t nseg,
                                 const int *__restrict__ cnt, const int *__restrict__ nxt, int64_t *__restrict__ ccnt,
                                 int *__restrict__ cnxt) {
  const int64_t nchunk = (nseg + kChunk - 1) / kChunk;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nchunk * kEntries;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ch = t / kEntries;
    int e = (int)(t % kEntries);
    int64_t total = 0;
    for (int64_t s = ch * kChunk; s < min(nseg, (ch + 1) * kChunk) && e >= 0; ++s) {
      int c, n;
      seg_step(consume, nraw, cnt, nxt, s, e, c, n);
      total += c;
      e = n;
    }
    ccnt[t] = total;
    cnxt[t] = e;
  }
}

// one thread: chunk entries and output bases
__global__ void chunk_scan_kernel(const uint8_t *__restrict__ consume, int64_t nraw, int64_t nseg,
                                  const int *__restrict__ cnt, const int *__restrict__ nxt,
                                  const int64_t *__restrict__ ccnt, const int *__restrict__ cnxt,
                                  int *__restrict__ centry, int64_t *__restrict__ cbase, int64_t nout,
                                  int *__restrict__ status) {
  if (threadIdx.x || blockIdx.x) return;
  const int64_t nchunk = (nseg + kChunk - 1) / kChunk;
  int e = 0;
  int64_t base = 0;
  for (int64_t ch = 0; ch < nchunk; ++ch) {
    centry[ch] = e;
    cbase[ch] = base;
    if (base >= nout || e < 0) {
      centry[ch] = -1;
      continue;
    }
    if (e < kEntries) {
      base += ccnt[ch * kEntries + e];
      e = cnxt[ch * kEntries + e];
    } else {
      for (int64_t s = ch * kChunk; s < min(nseg, (ch + 1) * kChunk) && e >= 0; ++s) {
        int c, n;
        seg_step(consume, nraw, cnt, nxt, s, e, c, n);
        base += c;
        e = n;
      }
    }
  }
  *status = base >= nout ? 0 : 1;  // 1: more words needed
}

// per chunk: segment entries and bases; then per segment: write the outputs
__global__ void seg_scan_kernel(const uint8_t *__restrict__ consume, int64_t nraw, int64_t nseg,
                                const int *__restrict__ cnt, const int *__restrict__ nxt,
                                const int *__restrict__ centry, const int64_t *__restrict__ cbase,
                                int *__restrict__ sentry, int64_t *__restrict__ sbase) {
  const int64_t nchunk = (nseg + kChunk - 1) / kChunk;
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunk;
       ch += (int64_t)gridDim.x * blockDim.x) {
    int e = centry[ch];
    int64_t base = cbase[ch];
    for (int64_t s = ch * kChunk; s < min(nseg, (ch + 1) * kChunk); ++s) {
      sentry[s] = e;
      sbase[s] = base;
      if (e < 0) continue;
      int c, n;
      seg_step(consume, nraw, cnt, nxt, s, e, c, n);
      base += c;
      e = n;
    }
  }
}

__global__ void emit_kernel(const uint8_t *__restrict__ consume, const double *__restrict__ value,
                            const uint8_t *__restrict__ tail, const uint64_t *__restrict__ raw, int64_t nraw,
                            int64_t nseg, const int *__restrict__ sentry, const int64_t *__restrict__ sbase,
                            double *__restrict__ out, int64_t nout, int64_t *__restrict__ tail_rec,
                            uint64_t *__restrict__ tail_words, int *__restrict__ ntail, int max_tail) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int e = sentry[s];
    if (e < 0) continue;
    int64_t pos = s * kSeg + e, o = sbase[s];
    const int64_t end = (s + 1) * kSeg;
    while (pos < end && pos < nraw && o < nout) {
      out[o] = value[pos];
      if (tail[pos]) {
        const int slot = atomicAdd(ntail, 1);
        if (slot < max_tail) {
          tail_rec[2 * slot] = o;
          tail_rec[2 * slot + 1] = pos;  // word position of the draw (its r; the accepted pair follows)
          for (int q = 0; q < kTailWords; ++q) tail_words[(int64_t)slot * kTailWords + q] = pos + q < nraw ? raw[pos + q] : 0;
        }
      }
      pos += consume[pos];
      ++o;
    }
  }
}

__global__ void scatter_kernel(const int64_t *__restrict__ idx, const double *__restrict__ v, int n,
                               double *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[idx[t]] = v[t];
}

struct OmegaWs {
  uint64_t *raw;
  uint8_t *consume, *tail;
  double *value;
  int *cnt, *nxt, *cnxt, *centry, *sentry, *ntail, *status;
  int64_t *ccnt, *cbase, *sbase, *tail_rec;
  uint64_t *tail_words;
  double *tail_val;
  int64_t nraw, nseg, nchunk;
  int max_tail;
};

OmegaWs carve_omega(Arena &ar, int64_t n, int64_t w) {
  OmegaWs o;
  const int64_t nout = n * w;
  o.nraw = round_up(nout + nout / 32 + 4096, kSeg);  // ~0.9 % of draws take extra words
  o.nseg = o.nraw / kSeg;
  o.nchunk = ceil_div(o.nseg, kChunk);
  o.max_tail = (int)std::min<int64_t>(std::max<int64_t>(4096, nout / 256), 1 << 22);
  o.raw = ar.take<uint64_t>(o.nraw);
  o.value = ar.take<double>(o.nraw);
  o.consume = ar.take<uint8_t>(o.nraw);
  o.tail = ar.take<uint8_t>(o.nraw);
  o.cnt = ar.take<int>(o.nseg * kEntries);
  o.nxt = ar.take<int>(o.nseg * kEntries);
  o.ccnt = ar.take<int64_t>(o.nchunk * kEntries);
  o.cnxt = ar.take<int>(o.nchunk * kEntries);
  o.centry = ar.take<int>(o.nchunk);
  o.cbase = ar.take<int64_t>(o.nchunk);
  o.sentry = ar.take<int>(o.nseg);
  o.sbase = ar.take<int64_t>(o.nseg);
  o.tail_rec = ar.take<int64_t>(2 * (int64_t)o.max_tail);
  o.tail_words = ar.take<uint64_t>((int64_t)o.max_tail * kTailWords);
  o.tail_val = ar.take<double>(o.max_tail);
  o.ntail = ar.take<int>(4);
  o.status = ar.take<int>(4);
  return o;
}

}  // namespace

size_t omega_ws_bytes(int64_t n, int64_t w) {
  Arena ar;
  ar.dry = true;
  carve_omega(ar, n, w);
  return ar.off + 1024;
}

// Omega (n x w, row-major fp64) for the Philox key of SeedSequence([seed, 0x534B, n, w]).
// Synchronises the stream (tail values are finished on the host).
int omega_device(uint64_t key0, uint64_t key1, int64_t n, int64_t w, double *out, void *ws, size_t ws_bytes,
                 cudaStream_t st) {
  if (n < 1 || w < 1) return fail(LRAMM_ERR_SHAPE, "omega: empty shape");
  Arena ar(ws, ws_bytes);
  OmegaWs o = carve_omega(ar, n, w);
  if (!ar.ok()) return fail(LRAMM_ERR_WORKSPACE, "omega: workspace too small");
  const int64_t nout = n * w;
  const int g = 8 * num_sms();
  philox_kernel<<<g, 256, 0, st>>>(o.raw, o.nraw, key0, key1);
  attempt_kernel<<<g, 256, 0, st>>>(o.raw, o.nraw, o.consume, o.value, o.tail);
  seg_map_kernel<<<g, 256, 0, st>>>(o.consume, o.nraw, o.nseg, o.cnt, o.nxt);
  chunk_map_kernel<<<(unsigned)ceil_div(o.nchunk * kEntries, 128), 128, 0, st>>>(o.consume, o.nraw, o.nseg, o.cnt,
                                                                                  o.nxt, o.ccnt, o.cnxt);
  chunk_scan_kernel<<<1, 32, 0, st>>>(o.consume, o.nraw, o.nseg, o.cnt, o.nxt, o.ccnt, o.cnxt, o.centry, o.cbase,
                                      nout, o.status);
  seg_scan_kernel<<<(unsigned)ceil_div(o.nchunk, 128), 128, 0, st>>>(o.consume, o.nraw, o.nseg, o.cnt, o.nxt,
                                                                    o.centry, o.cbase, o.sentry, o.sbase);
  LRAMM_CUDA_TRY(cudaMemsetAsync(o.ntail, 0, sizeof(int), st));
  emit_kernel<<<(unsigned)ceil_div(o.nseg, 128), 128, 0, st>>>(o.consume, o.value, o.tail, o.raw, o.nraw, o.nseg,
                                                                o.sentry, o.sbase, out, nout, o.tail_rec,
                                                                o.tail_words, o.ntail, o.max_tail);
  LRAMM_LAUNCH_CHECK();
  int hs[2] = {0, 0};
  LRAMM_CUDA_TRY(cudaMemcpyAsync(&hs[0], o.status, sizeof(int), cudaMemcpyDeviceToHost, st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(&hs[1], o.ntail, sizeof(int), cudaMemcpyDeviceToHost, st));
  LRAMM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hs[0]) return fail(LRAMM_ERR_NONCONVERGENCE, "omega: generated word stream too short");
  if (hs[1] > o.max_tail) return fail(LRAMM_ERR_WORKSPACE, "omega: too many tail draws");
  if (hs[1] == 0) return LRAMM_OK;
  // tail draws: recompute R + xx with the host libm's log1p (NumPy's npy_log1p)
  const int nt = hs[1];
  std::vector<int64_t> rec(2 * (size_t)nt);
  std::vector<uint64_t> words((size_t)nt * kTailWords);
  LRAMM_CUDA_TRY(cudaMemcpyAsync(rec.data(), o.tail_rec, rec.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LRAMM_CUDA_TRY(
      cudaMemcpyAsync(words.data(), o.tail_words, words.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  LRAMM_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<double> vals(nt);
  std::vector<int64_t> idx(nt);
  for (int t = 0; t < nt; ++t) {
    // the whole draw again, from its first word (earlier attempts may have been rejected)
    const uint64_t *wd = &words[(size_t)t * kTailWords];
    bool done = false;
    double v = 0.0;
    int j = 0;
    while (!done && j < kTailWords) {
      uint64_t r = wd[j++];
      const int zi = (int)(r & 0xFF);
      r >>= 8;
      const int sign = (int)(r & 1);
      const uint64_t rabs = (r >> 1) & 0x000FFFFFFFFFFFFFULL;
      double x = (double)rabs * kZigWHost[zi];
      if (sign) x = -x;
      if (rabs < kZigKHost[zi]) {
        v = x;
        done = true;
        break;
      }
      if (zi == 0) {
        while (j + 1 < kTailWords) {
          const double u1 = (double)(wd[j] >> 11) * (1.0 / 9007199254740992.0);
          const double u2 = (double)(wd[j + 1] >> 11) * (1.0 / 9007199254740992.0);
          j += 2;
          const double xx = -kZigInvR * std::log1p(-u1);
          const double yy = -std::log1p(-u2);
          if (yy + yy > xx * xx) {
            v = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
            done = true;
            break;
          }
        }
        break;
      }
      if (j >= kTailWords) break;
      const double u = (double)(wd[j++] >> 11) * (1.0 / 9007199254740992.0);
      if ((kZigFHost[zi - 1] - kZigFHost[zi]) * u + kZigFHost[zi] < std::exp(-0.5 * x * x)) {
        v = x;
        done = true;
      }
    }
    if (!done) return fail(LRAMM_ERR_NONCONVERGENCE, "omega: tail draw longer than %d words", kTailWords);
    vals[t] = v;
    idx[t] = rec[2 * t];
  }
  // scatter the corrected values (one small upload + kernel)
  double *dv = o.tail_val;
  int64_t *di = o.tail_rec;  // reuse: indices
  LRAMM_CUDA_TRY(cudaMemcpyAsync(dv, vals.data(), nt * sizeof(double), cudaMemcpyHostToDevice, st));
  LRAMM_CUDA_TRY(cudaMemcpyAsync(di, idx.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  scatter_kernel<<<(unsigned)ceil_div(nt, 256), 256, 0, st>>>(di, dv, nt, out);
  LRAMM_LAUNCH_CHECK();
  LRAMM_CUDA_TRY(cudaStreamSynchronize(st));
  return LRAMM_OK;
}

}  // namespace lramm
