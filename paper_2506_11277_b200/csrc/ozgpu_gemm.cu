// tcgen05 kind::i8 pair GEMMs of the B200-native Ozaki-I FP64 GEMM
// (replaces integer_gemm, proj/src/mma_sim.cpp:76-114, and the levelled
// accumulation, proj/src/scheme.cpp:314-355).
//
// Persistent, warp-specialised, one 128 x 256 output tile per work unit:
//   warp 0      TMA producer (3-D tensor maps over the [slice][row][kp] int8
//               slices, 128-byte swizzle, 4-stage mbarrier ring)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::i8
//               (M=128, N=256, K=32) into a double-buffered int32 TMEM
//               accumulator (2 x 256 columns)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue (TMEM lane quadrant = warp % 4)
//
// A "chunk" is a run of pairs on one diagonal whose int32 sum cannot
// overflow; its K loop runs over the concatenated slices (pairs x kp).
//
// Two epilogue modes:
//   split  (W == 0)  unit = (tile, chunk); the int32 chunk sum is written to
//                    plane[chunk] and a separate combine kernel rounds.
//   fused  (W = 2,3) unit = tile; the CTA walks every chunk of the tile and
//                    the epilogue folds each chunk sum, shifted by its
//                    diagonal weight, into a W-word exact integer per element
//                    kept in a CTA-private scratch (L2-resident); after the
//                    last chunk it rounds once (ExactValue::to_double,
//                    oracle.cpp:157-180) and stores C through an XOR-swizzled
//                    smem transpose so each warp writes whole rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "ozgpu_internal.h"
#include "ozgpu_numeric.h"
#include "ozgpu_ptx.cuh"

namespace ozgpu {

constexpr int kBN = 256;
constexpr int kStages = 4;  // 1-CTA kernel default (template parameter)
constexpr int kABytes = kBlockM * kBlockK;  // 16 KB
constexpr int kBBytes = kBN * kBlockK;      // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 2 * kBN;  // double-buffered accumulator
constexpr int kGemmThreads = 256;
constexpr int kStagingBytes = 4 * 32 * 32 * 8;  // fused epilogue: 32x32 f64 per warp
constexpr int kSmemSplit = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kSmemFused = kSmemSplit + kStagingBytes;

int gemm_smem_bytes() { return kSmemFused; }

struct TileCoord {
  int tm, tn;
};

// Grouped rasterisation: consecutive tiles walk 8 tile-rows at a time so
// concurrently running CTAs share A and B slice panels in L2.
__device__ __forceinline__ TileCoord decode_tile(int t, const GemmArgs& p) {
  const int G = p.group > 0 ? p.group : 8;
  const int group_size = G * p.tiles_n;
  const int group = t / group_size;
  const int first_m = group * G;
  const int gsz = p.tiles_m - first_m < G ? p.tiles_m - first_m : G;
  const int in_group = t - group * group_size;
  TileCoord c;
  c.tm = first_m + in_group % gsz;
  c.tn = in_group / gsz;
  return c;
}

// Chunk id at position `pos` of the unit's chunk sequence (proc_order
// permutes chunks so each bin's chunks are contiguous; null = identity).
__device__ __forceinline__ int chunk_at(const GemmArgs& p, int pos) {
  return p.proc_order ? __ldg(p.proc_order + pos) : pos;
}

// Work unit -> (tile, first chunk position, chunk count, linear tile index).
// Split mode: unit = (bin, tile), bin-major.  A bin is a run of chunks of
// one tile (bin_first[b] .. bin_first[b+1]) whose pair counts add up to the
// same total for every bin (host bin packing), so every CTA of a wave
// streams the same slice pair at the same time and shares it through L2.
__device__ __forceinline__ void decode_unit(int unit, const GemmArgs& p, bool fused,
                                            TileCoord& tc, int& c0, int& nc, int& tile,
                                            int mc_rank = -1) {
  if (mc_rank >= 0) {
    // 2-CTA cluster: unit = (bin, 256 x 256 super-tile); the CTA of rank r
    // takes its 128-row half (the two share the B panel through multicast)
    GemmArgs q = p;
    q.tiles_m = (p.tiles_m + 1) / 2;
    const int tiles = q.tiles_m * p.tiles_n;
    const int pos = unit / tiles;
    if (p.bin_first) {
      c0 = __ldg(p.bin_first + pos);
      nc = __ldg(p.bin_first + pos + 1) - c0;
    } else {
      c0 = pos;
      nc = 1;
    }
    tile = unit - pos * tiles;
    tc = decode_tile(tile, q);
    tc.tm = 2 * tc.tm + mc_rank;
    return;
  }
  if (fused) {
    tile = unit;
    tc = decode_tile(unit, p);
    c0 = 0;
    nc = p.nchunks;
  } else {
    const int tiles = p.tiles_m * p.tiles_n;
    const int pos = unit / tiles;
    if (p.bin_first) {
      c0 = __ldg(p.bin_first + pos);
      nc = __ldg(p.bin_first + pos + 1) - c0;
    } else {
      c0 = pos;
      nc = 1;
    }
    tile = unit - pos * tiles;
    if (p.pair_order) {
      // diagnostic: walk 256-row pair tiles (as the CTA-pair kernel does),
      // the two 128-row halves on consecutive units / CTAs
      GemmArgs q = p;
      q.tiles_m = p.tiles_m / 2;
      tc = decode_tile(tile >> 1, q);
      tc.tm = 2 * tc.tm + (tile & 1);
    } else {
      tc = decode_tile(tile, p);
    }
    if (p.dbg & 1) tc.tm = tc.tn = 0;  // experiment: every unit on tile 0 (results invalid)
  }
}
__device__ __forceinline__ void decode_unit(int unit, const GemmArgs& p, bool fused,
                                            TileCoord& tc, int& c0, int& nc, int mc_rank = -1) {
  int tile;
  decode_unit(unit, p, fused, tc, c0, nc, tile, mc_rank);
}

// Split-k tail: virtual unit -> (real unit, k-block range, partial?).
__device__ __forceinline__ bool tail_range(int& unit, const GemmArgs& p, int& kb0, int& kb1) {
  kb0 = 0;
  kb1 = p.kblocks;
  if (p.tail_parts == 0 || unit < p.tail_first) return false;
  const int v = unit - p.tail_first;
  const int r = v / p.tail_parts, part = v - r * p.tail_parts;
  unit = p.tail_first + r;
  kb0 = part * p.kblocks / p.tail_parts;
  kb1 = (part + 1) * p.kblocks / p.tail_parts;
  return true;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}
// Wave lockstep (see GemmArgs::sync): called by the whole producer warp at
// every k-step; returns the (warp-uniform) new lockstep state.  CTAs of a
// wave share their operand panels through L2 only while they stream them at
// about the same time, and a deep TMA pipeline hides exactly the misses that
// would otherwise keep them together -- measured on B200, the drift doubles
// or triples DRAM reads.  Every sync_g k-steps the cluster publishes its
// group and waits until all clusters have passed the group sync_d back.
__device__ __forceinline__ int ld_relaxed_gpu(const int* ptr) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}
// `seen` carries a prefetched read of the next wait slot: it is issued half
// a group early so that, in the common case, the check at the boundary costs
// no round trip and the producer keeps its ring full.
__device__ __forceinline__ bool lockstep_point(const GemmArgs& p, int step, bool lockstep,
                                               int& seen) {
  if (!lockstep) return false;
  const int r = step % p.sync_g;
  if (p.sync_prefetch && r == p.sync_g / 2 && r != 0) {  // prefetch the next boundary's slot
    const int hgrp = step / p.sync_g + 1 - p.sync_d;
    if (hgrp >= 0 && elect_one()) seen = ld_relaxed_gpu(p.sync + (hgrp & 63) * 32);
    __syncwarp();
    return true;
  }
  if (r != 0) return true;
  if (step >= p.sync_steps) return false;
  const int g = step / p.sync_g;
  if (elect_one()) {
    atomicAdd(p.sync + (g & 63) * 32, 1);  // one 128-byte line per slot
    const int hgrp = g - p.sync_d;
    if (hgrp >= 0) {
      const int target = (hgrp / 64 + 1) * p.sync_clusters;
      const int* slot = p.sync + (hgrp & 63) * 32;
      if (seen < target) {
        long long spins = 0;
        while (ld_acquire_gpu(slot) < target) {
          __nanosleep(64);
          if (++spins > (1 << 16)) {  // ~50 ms: a cluster is not resident; stop syncing
            lockstep = false;
            break;
          }
        }
      }
    }
    seen = -1;
  }
  return __all_sync(0xFFFFFFFFu, lockstep);
}

__device__ __forceinline__ void epilogue_bar() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// Final-chunk epilogue of the split+final mode: for one 32-column slab of the
// warp's 32 rows, sum every chunk of the tile diagonal by diagonal (the final
// chunk from TMEM registers, the others from their int32 planes), Horner-
// accumulate V = V * 2^t + S_d in 128 bits, round once (round_i128) and stage
// the doubles for a row-coalesced store.
__device__ __forceinline__ void final_combine_slab(const GemmArgs& p, const uint32_t (&r)[32],
                                                   int row, int col0, long qrow, int lane,
                                                   double* stage_w) {
  const int qcol = col0 + lane < p.n ? __ldg(p.qb + col0 + lane) : 0;
  const bool row_ok = row < p.m;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int cb = col0 + half * 16;
    const bool full16 = cb + 16 <= p.n;
    unsigned __int128 v[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) v[jj] = 0;
    for (int d = 0; d < p.diagonals; ++d) {
      long long s[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) s[jj] = 0;
      const int c_end = __ldg(p.diag_first + d + 1);
      for (int c = __ldg(p.diag_first + d); c < c_end; ++c) {
        if (c == p.final_chunk) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) s[jj] += static_cast<int32_t>(r[half * 16 + jj]);
        } else if (row_ok) {
          const int32_t* src = p.planes + static_cast<int64_t>(c) * p.plane_stride +
                               static_cast<int64_t>(row) * p.ldp + cb;
          if (full16) {
            const int4* s4 = reinterpret_cast<const int4*>(src);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int4 x = __ldcg(s4 + u);
              s[4 * u] += x.x;
              s[4 * u + 1] += x.y;
              s[4 * u + 2] += x.z;
              s[4 * u + 3] += x.w;
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
              if (cb + jj < p.n) s[jj] += __ldcg(src + jj);
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)
        v[jj] = (v[jj] << p.width) + static_cast<unsigned __int128>(static_cast<__int128>(s[jj]));
    }
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = half * 16 + jj;
      const int qj = __shfl_sync(0xFFFFFFFFu, qcol, j);
      stage_w[lane * 32 + (j ^ lane)] = round_i128(v[jj], qrow + qj + p.w_last);
    }
  }
}

// Row-coalesced store of a staged 32x32 block of C (optionally D = a*C + b*Cin).
__device__ __forceinline__ void store_staged(const GemmArgs& p, const double* stage_w, int row0,
                                             int col0, int lane) {
  __syncwarp();
  const int col = col0 + lane;
#pragma unroll 4
  for (int rr = 0; rr < 32; ++rr) {
    const int orow = row0 + rr;
    double d = stage_w[rr * 32 + (lane ^ rr)];
    if (orow < p.m && col < p.n) {
      if (p.axpby)
        d = __dadd_rn(__dmul_rn(p.alpha, d),
                      __dmul_rn(p.beta, p.cin[static_cast<int64_t>(orow) * p.ldcin + col]));
      p.c[static_cast<int64_t>(orow) * p.ldc + col] = d;
    }
  }
  __syncwarp();
}

// MC: launched as 2-CTA clusters; the two CTAs compute vertically adjacent
// 128 x 256 tiles with the same B panel, each loading half of every B stage
// and multicasting it to both (L2 -> SM operand traffic 64 KB instead of
// 96 KB per 2 x 128 x 256 x 128 step).  A stage is refilled only after both
// CTAs' MMAs released it (empty barriers count 2, commits multicast).
template <int W, bool MC, int kStages = 4>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   const GemmArgs p) {
  constexpr bool kFused = W >= 2;
  constexpr bool kFinal = W == 1;
  static_assert(!MC || W == 0, "multicast is a split-mode variant");
  const int mc_rank = MC ? static_cast<int>(cluster_ctarank()) : -1;
  const int unit0 = MC ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int ustep = MC ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  double* staging = reinterpret_cast<double*>(smem + kStages * kStageBytes + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
  }
  if (warp == 2) tmem_alloc(tmem_holder, kTmemCols);
  tc_fence_before();
  if constexpr (MC)
    cluster_sync();  // the peer's barriers exist before any multicast lands
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer (warp-wide loop, one elected issuer) ----------------
    int stage = 0;
    uint32_t phase = 0;
    int step = 0;
    bool lockstep = p.sync != nullptr && mc_rank <= 0;
    int seen = -1;
    for (int unit = unit0; unit < p.total_units; unit += ustep) {
      TileCoord tc;
      int c0, nc;
      decode_unit(unit, p, kFused, tc, c0, nc, mc_rank);
      for (int c = c0; c < c0 + nc; ++c) {
        const ChunkDesc cd = p.chunks[chunk_at(p, c)];
        for (int pr = 0; pr < cd.npairs; ++pr) {
          const int l = cd.l0 + pr;
          const int h = cd.d + 2 - l;
          for (int kb = 0; kb < p.kblocks; ++kb, ++step) {
            lockstep = lockstep_point(p, step, lockstep, seen);
            mbar_wait(&empty[stage], phase ^ 1);
            if (elect_one()) {
              mbar_expect_tx(&full[stage], kStageBytes);
              tma_load_3d(sA + stage * kABytes, &tma, &full[stage], kb * kBlockK,
                          tc.tm * kBlockM, l - 1);
              if constexpr (MC)
                tma_load_3d_mc(sB + stage * kBBytes + mc_rank * (kBBytes / 2), &tmb,
                               &full[stage], kb * kBlockK, tc.tn * kBN + mc_rank * (kBN / 2),
                               h - 1, 3);
              else
                tma_load_3d(sB + stage * kBBytes, &tmb, &full[stage], kb * kBlockK,
                            tc.tn * kBN, h - 1);
            }
            __syncwarp();
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-wide loop, one elected issuer) ----------------
    constexpr uint32_t idesc = idesc_i8<kBlockM, kBN>();
    const uint64_t ad0 = sdesc_sw128(smem_addr(sA));
    const uint64_t bd0 = sdesc_sw128(smem_addr(sB));
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int unit = unit0; unit < p.total_units; unit += ustep) {
      TileCoord tc;
      int c0, nc;
      decode_unit(unit, p, kFused, tc, c0, nc, mc_rank);
      for (int c = c0; c < c0 + nc; ++c, ++it) {
        const ChunkDesc cd = p.chunks[chunk_at(p, c)];
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * kBN;
        const int total = cd.npairs * p.kblocks;
        for (int i = 0; i < total; ++i) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            // descriptor start addresses advance in 16-byte units
            const uint64_t ad = ad0 + static_cast<uint64_t>(stage * (kABytes >> 4));
            const uint64_t bd = bd0 + static_cast<uint64_t>(stage * (kBBytes >> 4));
#pragma unroll
            for (int kk = 0; kk < kBlockK / 32; ++kk)
              tc_mma_i8(tmem_d, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0);
            if constexpr (MC)
              tc_commit_mc(&empty[stage], 3);
            else
              tc_commit(&empty[stage]);
            if (i == total - 1) tc_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    double* stage_w = staging + q * 32 * 32;
    uint64_t* scratch = nullptr;
    if constexpr (kFused)
      scratch = p.scratch + static_cast<size_t>(blockIdx.x) * W * kBN * kBlockM;
    int it = 0;
    for (int unit = unit0; unit < p.total_units; unit += ustep) {
      TileCoord tc;
      int c0, nc, tile;
      decode_unit(unit, p, kFused, tc, c0, nc, tile, mc_rank);
      const int row0 = tc.tm * kBlockM + q * 32;
      const int row = row0 + lane;
      long qrow = 0;
      if constexpr (kFused || kFinal) qrow = row < p.m ? __ldg(p.qa + row) : 0;
      for (int cpos = c0; cpos < c0 + nc; ++cpos, ++it) {
        const int c = kFused ? cpos : chunk_at(p, cpos);
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kBN;
        if (kFinal && c == p.final_chunk) {
          // every other chunk of this tile must have stored its plane
          if (threadIdx.x == 128) {
            while (ld_acquire_gpu(p.tile_counters + tile) < p.nchunks - 1) __nanosleep(200);
            __threadfence();
          }
          epilogue_bar();
#pragma unroll 1
          for (int s0 = 0; s0 < kBN; s0 += 32) {
            uint32_t r[32];
            tmem_ld32(taddr + s0, r);
            const int col0 = tc.tn * kBN + s0;
            final_combine_slab(p, r, row, col0, qrow, lane, stage_w);
            store_staged(p, stage_w, row0, col0, lane);
          }
        } else if constexpr (!kFused) {
          int32_t* dst = p.planes + static_cast<int64_t>(c) * p.plane_stride +
                         static_cast<int64_t>(row) * p.ldp;
#pragma unroll 1
          for (int s0 = 0; s0 < kBN; s0 += 32) {
            uint32_t r[32];
            tmem_ld32(taddr + s0, r);
            const int col0 = tc.tn * kBN + s0;
            if (row < p.m) {
              if (col0 + 32 <= p.n && (p.ldp & 3) == 0) {
                int4* d4 = reinterpret_cast<int4*>(dst + col0);
#pragma unroll
                for (int v = 0; v < 8; ++v)
                  d4[v] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
              } else {
                for (int v = 0; v < 32; ++v)
                  if (col0 + v < p.n) dst[col0 + v] = static_cast<int32_t>(r[v]);
              }
            }
          }
          if constexpr (kFinal) {
            // publish this chunk of the tile (release: fence by every writer,
            // then one counter increment after the epilogue barrier)
            __threadfence();
            epilogue_bar();
            if (threadIdx.x == 128) atomicAdd(p.tile_counters + tile, 1);
          }
        } else {
          const bool first = c == 0, last = c == p.nchunks - 1;
          const int shift = p.chunks[c].shift;
#pragma unroll 1
          for (int s0 = 0; s0 < kBN; s0 += 32) {
            uint32_t r[32];
            tmem_ld32(taddr + s0, r);
            // scratch layout [word][column][row]: a warp touches 256 contiguous bytes
            uint64_t* sp = scratch + static_cast<size_t>(s0) * kBlockM + q * 32 + lane;
            const int col0 = tc.tn * kBN + s0;
            int qcol = 0;
            if (last) qcol = col0 + lane < p.n ? __ldg(p.qb + col0 + lane) : 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              uint64_t v[W];
#pragma unroll
              for (int w = 0; w < W; ++w)
                v[w] = first ? 0ULL : sp[(static_cast<size_t>(w) * kBN + j) * kBlockM];
              words_add_shifted<W>(v, static_cast<int32_t>(r[j]), shift);
              const int qj = __shfl_sync(0xFFFFFFFFu, qcol, j);
              if (!last) {
#pragma unroll
                for (int w = 0; w < W; ++w) sp[(static_cast<size_t>(w) * kBN + j) * kBlockM] = v[w];
              } else {
                const double d = round_words<W>(v, qrow + qj + p.w_last);
                stage_w[lane * 32 + (j ^ lane)] = d;
              }
            }
            if (last) store_staged(p, stage_w, row0, col0, lane);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
  }

  tc_fence_before();
  if constexpr (MC)
    cluster_sync();  // no CTA leaves while its peer may still multicast into it
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ----------------------------------------------------------------------------
// CTA-pair variant (split mode): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile with tcgen05.mma.cta_group::2 (M=256, N=256, K=32) issued by
// the leader CTA.  Each CTA stages its own 128 A rows and 128 of the 256 B
// rows per k-block (32 KB / stage, 6 stages), so per-SM operand traffic from
// L2 drops from 48 KB to 32 KB per 128x256x128 of work versus the 1-CTA tile.
// The peers' TMA transactions land on the leader's full barrier; the
// leader's commits multicast to both CTAs' empty / tmem-full barriers; the
// epilogue warps of both CTAs release the accumulator on the leader.
// ----------------------------------------------------------------------------

constexpr int kPairHalfBytes = 128 * kBlockK;             // 16 KB (A or B half)
// per-CTA stage bytes for a 256 x kPN pair tile: A 128 rows + B kPN / 2 rows
constexpr int pair_stage_bytes(int pn) { return kPairHalfBytes + (pn / 2) * kBlockK; }
// + the epilogue's TMA-store staging: 4 warps x 2 buffers x (32 x 32 int32)
constexpr int kPairCStage = 4 * 2 * 4096;
constexpr int smem_pair(int stages, int pn = 256) {
  return stages * pair_stage_bytes(pn) + kPairCStage + 1024 + 256;
}

// kPN = 256: 256 x 256 tiles, double-buffered 256-column accumulators.
// kPN = 512: 256 x 512 tiles (two N = 256 MMAs per K step into the two
// TMEM halves, single-buffered): 1.5x the operand bytes per stage for 2x
// the MMAs, so each wave of CTA pairs covers twice the C area per slice
// byte read (fewer DRAM and L2 -> SM bytes per int8 op).
// kCl = 4: clusters of two CTA pairs stacked in M (a 512 x kPN super-tile)
// sharing the B panel: each pair loads one of the two 256-row B boxes and
// multicasts it to the same-half CTA of the other pair, so L2 -> SM operand
// traffic per MMA drops by a third; a stage is released only when both
// pairs' MMAs have consumed it (empty barriers count both commits).
template <int kPairStages, int kPN = 256, int kCl = 2>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_i8_pair_kernel(const __grid_constant__ CUtensorMap tma,
                        const __grid_constant__ CUtensorMap tmb,
                        const __grid_constant__ CUtensorMap tmc, const GemmArgs p) {
  static_assert(kPN == 256 || kPN == 512, "pair tile width");
  static_assert(kCl == 2 || (kCl == 4 && kPN == 512), "cluster shape");
  constexpr int kPairsPerCl = kCl / 2;
  constexpr int kRowsPerUnit = 256 * kPairsPerCl;
  constexpr int kHalves = kPN / 256;                // N = 256 MMAs per K step
  constexpr int kAcc = kPN == 256 ? 2 : 1;          // TMEM accumulators (512 columns in all)
  constexpr int kBStage = kHalves * kPairHalfBytes;  // this CTA's B rows per stage
  constexpr int kStage = kPairHalfBytes + kBStage;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kPairStages * kPairHalfBytes;
  uint32_t* cstage = reinterpret_cast<uint32_t*>(smem + kPairStages * kStage);  // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPairStages * kStage + kPairCStage);
  uint64_t* empty = full + kPairStages;
  uint64_t* tfull = empty + kPairStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t prk = crank >> 1;           // CTA pair within the cluster
  const uint32_t rank = crank & 1;           // CTA within the pair
  const uint32_t lead_rank = crank & ~1u;    // the pair leader's cluster rank
  const bool leader = rank == 0;             // pair leader: issues the MMAs
  const int pair = blockIdx.x / kCl;         // cluster index (work distribution)
  const int npairs = gridDim.x / kCl;
  constexpr uint16_t kEmptyMask = kCl == 4 ? 0xF : 0x3;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * prk));

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPairsPerCl);  // one commit per pair of the cluster
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
    if (p.tma_store)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmc)) : "memory");
  }
  if (warp == 2) tmem_alloc_pair(tmem_holder, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; warp-wide loop, elected issuer) ----------------
    const uint32_t full_leader0 = map_to_rank(&full[0], lead_rank);
    int stage = 0;
    uint32_t phase = 0;
    int step = 0;               // k-steps issued by this cluster
    bool lockstep = p.sync != nullptr && crank == 0;
    int seen = -1;
    for (int vunit = pair; vunit < p.total_units; vunit += npairs) {
      TileCoord tc;
      int c0, nc, kb0, kb1, unit = vunit;
      tail_range(unit, p, kb0, kb1);
      decode_unit(unit, p, false, tc, c0, nc);
      const int arow = tc.tm * kRowsPerUnit + static_cast<int>(prk) * 256 + static_cast<int>(rank) * 128;
      const int brow = tc.tn * kPN + static_cast<int>(rank) * 128;
      for (int c = c0; c < c0 + nc; ++c) {
      const ChunkDesc cd = p.chunks[chunk_at(p, c)];
      for (int pr = 0; pr < cd.npairs; ++pr) {
        const int l = cd.l0 + pr;
        const int h = cd.d + 2 - l;
        for (int kb = kb0; kb < kb1; ++kb, ++step) {
          lockstep = lockstep_point(p, step, lockstep, seen);
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            // (OZGPU_DBG bit 2, experiment: every B box is loaded twice)
            const int breps = (p.dbg & 4) ? 2 : 1;
            if (leader) mbar_expect_tx(&full[stage], 2 * (kPairHalfBytes + breps * kBStage));
            const uint32_t bar = full_leader0 + 8 * stage;
            if (p.l2_hint) {
              const uint64_t pol = p.l2_hint == 1 ? l2_policy_evict_last() : l2_policy_evict_normal();
              tma_load_3d_pair_hint(sA + stage * kPairHalfBytes, &tma, bar, kb * kBlockK, arow,
                                    l - 1, pol);
#pragma unroll
              for (int hh = 0; hh < kHalves; ++hh)
                tma_load_3d_pair_hint(sB + stage * kBStage + hh * kPairHalfBytes, &tmb, bar,
                                      kb * kBlockK, brow + hh * 256, h - 1, pol);
            } else if constexpr (kCl == 4) {
              tma_load_3d_pair(sA + stage * kPairHalfBytes, &tma, bar, kb * kBlockK, arow, l - 1);
              // this pair's B box (hh = prk) to the same-half CTA of both pairs
              tma_load_3d_pair_mc(sB + stage * kBStage + prk * kPairHalfBytes, &tmb, bar,
                                  kb * kBlockK, brow + static_cast<int>(prk) * 256, h - 1,
                                  static_cast<uint16_t>((1u << rank) | (1u << (rank + 2))));
            } else {
              tma_load_3d_pair(sA + stage * kPairHalfBytes, &tma, bar, kb * kBlockK, arow, l - 1);
              for (int rep = 0; rep < breps; ++rep)
#pragma unroll
                for (int hh = 0; hh < kHalves; ++hh)
                  tma_load_3d_pair(sB + stage * kBStage + hh * kPairHalfBytes, &tmb, bar,
                                   kb * kBlockK, brow + hh * 256, h - 1);
            }
          }
          __syncwarp();
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA; warp-wide loop, elected issuer) ----------------
    constexpr uint32_t idesc = idesc_i8<256, kBN>();
    const uint64_t ad0 = sdesc_sw128(smem_addr(sA));
    const uint64_t bd0 = sdesc_sw128(smem_addr(sB));
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int vunit = pair; vunit < p.total_units; vunit += npairs) {
      TileCoord tc;
      int c0, nc, kb0, kb1, unit = vunit;
      tail_range(unit, p, kb0, kb1);
      decode_unit(unit, p, false, tc, c0, nc);
      for (int c = c0; c < c0 + nc; ++c, ++it) {
      const ChunkDesc cd = p.chunks[chunk_at(p, c)];
      const int acc = it % kAcc;
      const uint32_t aphase = (it / kAcc) & 1;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * kPN;
      const int total = cd.npairs * (kb1 - kb0);
      int i0 = 0;
      if constexpr (kPN == 512) {
        // Single-buffered 512-column accumulator: the epilogue releases
        // columns 0-255 (tempty[0]) before 256-511 (tempty[1]).  Start the
        // chunk with the first ring's worth of k-steps on half 0 only, then
        // add their half-1 MMAs once half 1 is drained (the stages are
        // released by those later commits), so half 1's drain overlaps MMAs.
        const int lead = p.no_half_release ? 0 : (total < kPairStages ? total : kPairStages);
        if (p.no_half_release) {
          mbar_wait(&tempty[1], aphase ^ 1);
          tc_fence_after();
        }
        const int stage0 = stage;
        const uint32_t phase0 = phase;
        for (int i = 0; i < lead; ++i) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = ad0 + static_cast<uint64_t>(stage * (kPairHalfBytes >> 4));
            const uint64_t bd = bd0 + static_cast<uint64_t>(stage * (kBStage >> 4));
#pragma unroll
            for (int kk = 0; kk < kBlockK / 32; ++kk)
              tc_mma_i8_pair(tmem_d, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0);
          }
          __syncwarp();
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lead) {
          mbar_wait(&tempty[1], aphase ^ 1);
          tc_fence_after();
        }
        int st2 = stage0;
        (void)phase0;
        for (int i = 0; i < lead; ++i) {
          if (elect_one()) {
            const uint64_t ad = ad0 + static_cast<uint64_t>(st2 * (kPairHalfBytes >> 4));
            const uint64_t bd = bd0 + static_cast<uint64_t>(st2 * (kBStage >> 4));
#pragma unroll
            for (int kk = 0; kk < kBlockK / 32; ++kk)
              tc_mma_i8_pair(tmem_d + 256, ad + 2 * kk, bd + (kPairHalfBytes >> 4) + 2 * kk,
                             idesc, (i | kk) != 0);
            tc_commit_pair_mask(&empty[st2], kEmptyMask);
            if (i == total - 1) tc_commit_pair_mask(&tfull[acc], pair_mask);
          }
          __syncwarp();
          if (++st2 == kPairStages) st2 = 0;
        }
        i0 = lead;
      }
      for (int i = i0; i < total; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = ad0 + static_cast<uint64_t>(stage * (kPairHalfBytes >> 4));
          const uint64_t bd = bd0 + static_cast<uint64_t>(stage * (kBStage >> 4));
#pragma unroll
          for (int kk = 0; kk < kBlockK / 32; ++kk)
#pragma unroll
            for (int hh = 0; hh < kHalves; ++hh)
              tc_mma_i8_pair(tmem_d + hh * 256, ad + 2 * kk,
                             bd + hh * (kPairHalfBytes >> 4) + 2 * kk, idesc, (i | kk) != 0);
          tc_commit_pair_mask(&empty[stage], kEmptyMask);
          if (i == total - 1) tc_commit_pair_mask(&tfull[acc], pair_mask);
        }
        __syncwarp();
        if (++stage == kPairStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): TMEM -> int32 chunk plane ----------------
    const int q = warp & 3;
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], lead_rank);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], lead_rank);
    uint32_t* cbuf = cstage + q * 2 * 1024;  // this warp's two 32 x 32 int32 staging tiles
    int cb = 0;
    int it = 0;
    for (int vunit = pair; vunit < p.total_units; vunit += npairs) {
      TileCoord tc;
      int c0, nc, kb0, kb1, unit = vunit;
      const bool partial = tail_range(unit, p, kb0, kb1);
      decode_unit(unit, p, false, tc, c0, nc);
      for (int cpos = c0; cpos < c0 + nc; ++cpos, ++it) {
      const int c = chunk_at(p, cpos);
      const int acc = it % kAcc;
      const uint32_t aphase = (it / kAcc) & 1;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int row = tc.tm * kRowsPerUnit + static_cast<int>(prk) * 256 +
                      static_cast<int>(rank) * 128 + q * 32 + lane;
      int32_t* dst = p.planes + static_cast<int64_t>(c) * p.plane_stride +
                     static_cast<int64_t>(row) * p.ldp;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kPN;
#pragma unroll 1
      for (int s0 = 0; s0 < kPN; s0 += 32) {
        if (kPN == 512 && s0 == 256 && !p.no_half_release) {  // columns 0-255 drained: release half 0
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader0);
        }
        uint32_t r[32];
        tmem_ld32(taddr + s0, r);
        const int col0 = tc.tn * kPN + s0;
        if (p.tma_store && !(p.dbg & 2)) {
          // stage the warp's 32 rows x 32 columns in shared memory (128-byte
          // swizzle: conflict-free 16-byte writes) and let TMA write whole
          // lines -- a plain store for a full unit, an exact int32 reduce-add
          // for a split-k tail part; TMA clips rows >= m and columns >= n
          uint32_t* buf = cbuf + cb * 1024;
          if (lane == 0) bulk_wait_read<1>();  // the store that used `buf` has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int row0 = tc.tm * kRowsPerUnit + static_cast<int>(prk) * 256 +
                             static_cast<int>(rank) * 128 + q * 32;
            if (partial)
              tma_reduce_add_3d(&tmc, buf, col0, row0, c);
            else
              tma_store_3d(&tmc, buf, col0, row0, c);
            bulk_commit();
          }
          cb ^= 1;
        } else if (p.dbg & 2) {  // experiment: no plane stores (results invalid)
          if (r[0] == 0x7fffffffu && r[31] == 0x7fffffffu) dst[col0] = 0;
        } else if (row < p.m && partial) {  // exact integer partial sums: order-free
          for (int v = 0; v < 32; ++v)
            if (col0 + v < p.n && r[v] != 0u) atomicAdd(dst + col0 + v, static_cast<int>(r[v]));
        } else if (row < p.m) {
          if (col0 + 32 <= p.n && (p.ldp & 3) == 0) {
            int4* d4 = reinterpret_cast<int4*>(dst + col0);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              d4[v] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          } else {
            for (int v = 0; v < 32; ++v)
              if (col0 + v < p.n) dst[col0 + v] = static_cast<int32_t>(r[v]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      // kPN = 512: tempty[1] releases columns 256-511 (half 0 went above)
      if (lane == 0) {
        if (kPN == 512 && p.no_half_release) mbar_arrive_cluster(tempty_leader0);
        mbar_arrive_cluster((acc || kPN == 512) ? tempty_leader1 : tempty_leader0);
      }
      }
    }
  }

  if (warp >= 4 && p.tma_store && lane == 0) bulk_wait<0>();  // staged plane stores done
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

// cudaFuncSetAttribute is per device: remember which devices a kernel's
// dynamic shared-memory limit was raised on (bit per device ordinal).
__host__ inline bool needs_config(unsigned long long& done_mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ULL << (dev & 63);
  if (done_mask & bit) return false;
  done_mask |= bit;
  return true;
}

template <int S, int PN = 256, int CL = 2>
static cudaError_t launch_pair_t(const CUtensorMap* tma, const CUtensorMap* tmb,
                                 const CUtensorMap* tmc, const GemmArgs& args, int clusters,
                                 cudaStream_t st) {
  static unsigned long long configured = 0;
  if (needs_config(configured)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_pair_kernel<S, PN, CL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_pair(S, PN));
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL * clusters);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem_pair(S, PN);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_i8_pair_kernel<S, PN, CL>, *tma, *tmb, *tmc, args);
}

cudaError_t launch_gemm_i8_pair(const CUtensorMap* tma, const CUtensorMap* tmb,
                                const CUtensorMap* tmc, const GemmArgs& args, int num_sms,
                                cudaStream_t st, int64_t* launches) {
  const int cl = args.cluster_ctas == 4 ? 4 : 2;
  int pairs = args.max_clusters > 0 ? args.max_clusters : num_sms / cl;  // clusters
  if (args.total_units < pairs) pairs = args.total_units;
  if (pairs < 1) return cudaSuccess;
  const char* sv = std::getenv("OZGPU_PAIR_STAGES");
  cudaError_t e0;
  if (args.pair_n == 512 && cl == 4) {
    const int stages = sv ? std::atoi(sv) : 4;
    e0 = stages == 3 ? launch_pair_t<3, 512, 4>(tma, tmb, tmc, args, pairs, st)
                     : launch_pair_t<4, 512, 4>(tma, tmb, tmc, args, pairs, st);
  } else if (args.pair_n == 512) {  // 48 KB stages: 4 (default) or 3
    const int stages = sv ? std::atoi(sv) : 4;
    e0 = stages == 3 ? launch_pair_t<3, 512>(tma, tmb, tmc, args, pairs, st)
                     : launch_pair_t<4, 512>(tma, tmb, tmc, args, pairs, st);
  } else {
    const int stages = sv ? std::atoi(sv) : 6;
    e0 = stages >= 6 ? launch_pair_t<6>(tma, tmb, tmc, args, pairs, st)  // 7 no longer fits
       : stages == 5 ? launch_pair_t<5>(tma, tmb, tmc, args, pairs, st)
       : stages == 3 ? launch_pair_t<3>(tma, tmb, tmc, args, pairs, st)
                     : launch_pair_t<4>(tma, tmb, tmc, args, pairs, st);
  }
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

template <int W>
static cudaError_t launch_t(const CUtensorMap* tma, const CUtensorMap* tmb, const GemmArgs& args,
                            int grid, int smem, cudaStream_t st) {
  static unsigned long long configured = 0;
  if (needs_config(configured)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_kernel<W, false, 4>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  gemm_i8_kernel<W, false, 4><<<grid, kGemmThreads, smem, st>>>(*tma, *tmb, args);
  return cudaGetLastError();
}

template <int S>
static cudaError_t launch_mc_t(const CUtensorMap* tma, const CUtensorMap* tmb_half,
                               const GemmArgs& args, int clusters, cudaStream_t st) {
  constexpr int smem = S * kStageBytes + 1024 + 256;
  static unsigned long long configured = 0;
  if (needs_config(configured)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_kernel<0, true, S>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_i8_kernel<0, true, S>, *tma, *tmb_half, args);
}

cudaError_t launch_gemm_i8_mc(const CUtensorMap* tma, const CUtensorMap* tmb_half,
                              const GemmArgs& args, int num_sms, cudaStream_t st,
                              int64_t* launches) {
  int clusters = num_sms / 2;
  if (args.total_units < clusters) clusters = args.total_units;
  if (clusters < 1) return cudaSuccess;
  const char* sv = std::getenv("OZGPU_MC_STAGES");
  const int stages = sv ? std::atoi(sv) : 4;
  cudaError_t e = stages == 3 ? launch_mc_t<3>(tma, tmb_half, args, clusters, st)
                              : launch_mc_t<4>(tma, tmb_half, args, clusters, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_gemm_i8(const CUtensorMap* tma, const CUtensorMap* tmb, const GemmArgs& args,
                           int num_sms, cudaStream_t st, int64_t* launches) {
  const int grid = args.total_units < num_sms ? args.total_units : num_sms;
  if (grid < 1) return cudaSuccess;
  cudaError_t e;
  switch (args.fused_words) {
    case 0: e = launch_t<0>(tma, tmb, args, grid, kSmemSplit, st); break;
    case 1: e = launch_t<1>(tma, tmb, args, grid, kSmemFused, st); break;
    case 2: e = launch_t<2>(tma, tmb, args, grid, kSmemFused, st); break;
    case 3: e = launch_t<3>(tma, tmb, args, grid, kSmemFused, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ozgpu
