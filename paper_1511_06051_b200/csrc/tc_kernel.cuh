// Persistent warp-specialised tcgen05 TF32 GEMM kernel (see conv_tc.cu for the operand
// modes and the host-side planners).
//
//   warps 0, 3  TMA producers (A / B operand): fill a `stages`-deep SMEM ring, one stage
//               per K block, with division-free incremental coordinates
//   warp 1      MMA issuer: tcgen05.mma.kind::tf32 into one of two TMEM accumulators
//   warp 2      TMEM allocator (512 columns = 2 x 256 fp32 accumulators)
//   warps 4..7  epilogue: TMEM -> registers -> padded SMEM transpose -> coalesced
//               128-byte row stores (bias / ReLU / accumulate / split-K partials)
// CTAs are persistent (grid = #SMs); tile t of a CTA uses accumulator t % 2, so the
// epilogue of tile t overlaps the MMAs of tile t + 1.
#pragma once

#include "tc_gemm.cuh"

namespace psg {
namespace tck {

enum AMode { A_RECT_K = 0, A_2D_K = 1, A_RECT_MN = 2, A_2D_MN = 3, A_IM2COL_K = 4 };
enum BMode { B_2D_K = 0, B_WT_MN = 1, B_RECT_MN = 2, B_2D_MN = 3, B_COL_MN = 4, B_TAPS_MN = 5,
             B_3D_K = 6, B_TAPS_IM2COL = 7 };
enum RowMap { ROW_RECT = 0, ROW_LINEAR = 1 };

// Warp roles: 0..3 and 6..7 TMA producers (K block it -> producer it % p.producers),
// 4 MMA issuer, 5 TMEM allocator, 8..11 epilogue (warp % 4 selects the TMEM lane quarter).
constexpr int kMaxProducers = 6;
constexpr int kMmaWarp = 4, kAllocWarp = 5, kEpiWarp0 = 8;
constexpr int kThreads = 384;
constexpr int kTileM = 128;
constexpr int kAccCols = 256;                 // one accumulator: 128 lanes x 256 fp32
constexpr int kEpiBytes = 2 * kAccCols * 4;  // static smem: the bias of each accumulator's tile
// TMA-store epilogue staging: per epilogue warp one or two 32 x 32-float chunks
// (SWIZZLE_128B), 4 KB each
constexpr int kOutChunkBytes = 32 * 32 * 4;

struct TcArgs {
  int a_mode, b_mode, row_map;
  int n_tile;             // UMMA N (multiple of 16, <= 256)
  int stage_bytes, a_bytes, stages;  // stage_bytes: one K block's A + B (a "slot")
  int kps;                // K blocks per pipeline stage (slots per stage)
  int a_chunks;           // MN-major A: 32-row chunks actually loaded (M tail skipped)
  int producers;          // TMA producer warps (<= kMaxProducers)
  int a_tx;               // A bytes landing per stage (expect_tx)
  int m_tiles, n_tiles;   // per (group, tap)
  int G, taps;            // group / tap index g * taps + tap
  int kblocks, kb_per_split, splits;
  long long total_tiles;  // m_tiles * n_tiles * G * taps * splits
  // coordinate helpers
  int a_c_g;              // A channel / M offset per group
  int b_r_g;              // B row (K or N) offset per group
  int b_n_g;              // B N offset per group (rect MN)
  int cb;                 // K blocks per tap (rect-K A, W^T B)
  int kw, ph, pw, sign;   // tap shift: coord = origin + sign * (u - p)
  // M rectangles (ROW_RECT)
  int rm, wm, th, tw;
  int out_h, out_w;
  // K rectangles (A/B_RECT_MN)
  int rk, wk, kth, ktw;
  // epilogue
  float* out;
  float* ws;
  long long ws_stride;
  const float* bias;
  int relu, accumulate;
  int ldo;
  int m_valid;            // rows valid in M (per group), ROW_LINEAR
  int n_valid;            // columns valid in N (per group)
  int col_g, col_tap, row_g;
  // B_TAPS_MN (multi-tap wgrad): virtual N = ntaps x cpt columns (cpt = C/G rounded up to
  // 32); column vc -> tap vc / cpt, channel vc % cpt (valid below cgs); dW column tap*cgs + c
  int ntaps, cpt, cgs;
  int valid_cols;         // split-K reduce: dW row padding columns (>= Kf) zeroed
  int epi_vec;            // epilogue: float4 stores (16-byte aligned rows and column runs)
  // CTA pairs (cta_group::2, launched as 2-CTA clusters): a work unit is two vertically
  // adjacent 128-row tiles (CTA rank r takes tile 2u + r) sharing one MMA of M = 256; each
  // CTA loads its own A tile and half of the B tile (b_cols columns).
  int pair;
  int pair_policy;        // ConvGeom::tc_pair: 0 heuristic, 1 never, 2 whenever legal
  // producer cursor jump over the other producers' stages: D = (producers - 1) * kps K
  // blocks split into the cursors' mixed-radix digits (host-computed, no divisions per stage)
  int adv_kb, adv_c0, adv_tap, adv_tv, adv_tu, adv_w, adv_h, adv_b;
  // MN-major operand tiles as ONE TMA box (map viewed as [chunks][rows][32 floats]: the
  // 32-column chunks stacked in smem exactly as the per-chunk boxes would land) instead of
  // one box per 32-column chunk — TMA issue cost is per box
  int a_one, b_one;
  int m_units;            // M work units: m_tiles, or ceil(m_tiles / 2) for pairs
  int b_cols;             // B columns (N) loaded per CTA: n_tile, or n_tile / 2 for pairs
  // A_IM2COL_K: M = linear pixels (b, y, x) of an out_h x out_w traversal grid; a tile's
  // first pixel sits at (x + im_lw, y + im_lh) of the source, tap (u, v) adds offsets
  // (sign > 0 ? v : kw - 1 - v, sign > 0 ? u : kh - 1 - u)
  int kh, im_lw, im_lh;
  // dgrad with the consumer-side ReLU backward folded in: out = (mask > 0 ? acc : 0), mask
  // laid out like out (the ReLU's output = this conv's input), applied before accumulate
  const float* mask;
  // TMA-store epilogue (fprop / dgrad / linear, ROW_LINEAR, float4-aligned outputs): a warp's
  // 32 rows x 32 columns go through a swizzled smem chunk and one cp.async.bulk.tensor store
  // (map_o: out [rows][ldo], or the split-K workspace [splits][rows][ldo]) instead of 32
  // row-strided float4 runs per store instruction; partial column chunks keep direct stores
  // multi-tap wgrad with a spare 32-column chunk in its last N tile: that chunk is loaded
  // from a ones matrix (map_o in EPI 2 kernels), so its columns accumulate
  // sum_pixels dY[pixel][f] = dbias[f] (model.hpp:560) in the same MMAs; written to db
  // (one split) or to the split's bias partial row (db_part[split][F])
  int bias_chunk;          // virtual chunk index of the ones chunk, or 0
  float* db;
  float* db_part;
  int db_ld;               // F
  int epi_tma;             // 0, or the staging chunks per epilogue warp (1 or 2)
  int ring_bytes;          // stage ring bytes (the staging area follows, 1024-aligned)
  // PSG_TC_PROF=1: per-launch clock64 counters (rank-0 CTAs): [0] MMA-loop cycles, [1] MMA
  // warp waiting for a full stage, [2] ... for a free accumulator, [3] stages consumed,
  // [4] producer 0 waiting for an empty slot, [5] producer-0 loop cycles, [6] epilogue warp 0
  // waiting for a finished accumulator, [7] epilogue-warp-0 loop cycles; null = off
  unsigned long long* prof;
};

// Per-tile B_TAPS_MN chunk table: tap shift and channel offset of each 32-column chunk.
constexpr int kMaxBChunks = 8;
struct TapChunks {
  int dx[kMaxBChunks], dy[kMaxBChunks], c[kMaxBChunks];
};

struct Tile {
  int m, n, g, tap, split;
};

__device__ __forceinline__ Tile decode_tile(const TcArgs& p, long long t) {
  Tile r;
  r.n = static_cast<int>(t % p.n_tiles);
  t /= p.n_tiles;
  r.m = static_cast<int>(t % p.m_units);
  t /= p.m_units;
  const int gt = static_cast<int>(t % (p.G * p.taps));
  r.split = static_cast<int>(t / (p.G * p.taps));
  r.g = gt / p.taps;
  r.tap = gt % p.taps;
  return r;
}

// B_TAPS_MN: tap shift and channel offset of every 32-column chunk of this CTA's B tile.
__device__ __forceinline__ void tap_chunks(const TcArgs& p, const Tile& t, TapChunks& k,
                                           int rank) {
#pragma unroll
  for (int j = 0; j < kMaxBChunks; ++j) {
    const int vc = t.n * p.n_tile + rank * p.b_cols + 32 * j;
    const int tap = min(vc / p.cpt, p.ntaps - 1);  // chunks past the last tap: harmless reloads
    k.dy[j] = tap / p.kw - p.ph;
    k.dx[j] = tap % p.kw - p.pw;
    k.c[j] = p.bias_chunk && (vc >> 5) == p.bias_chunk ? -1 : p.b_n_g * t.g + vc % p.cpt;
  }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Incremental K-block cursor: coordinates advance without divisions in the loop.
struct KCursor {
  int kb;
  int t0, t1;      // rect-K A / W^T B: (channel-or-filter block, tap)
  int tu, tv;      // tap coordinates
  int kbi, koh, kow;  // K pixel rectangle (MN rect operands)
  __device__ __forceinline__ void init(const TcArgs& p, int kb0) {
    kb = kb0;
    if (p.cb) {
      t0 = kb0 % p.cb;
      t1 = kb0 / p.cb;
      tu = t1 / p.kw;
      tv = t1 % p.kw;
    }
    if (p.kth) {
      kbi = kb0 / (p.kth * p.ktw);
      const int r = kb0 % (p.kth * p.ktw);
      koh = (r / p.ktw) * p.rk;
      kow = (r % p.ktw) * p.wk;
    }
  }
  // jump D = (producers - 1) * kps K blocks (digits precomputed in TcArgs::adv_*)
  __device__ __forceinline__ void advance(const TcArgs& p) {
    kb += p.adv_kb;
    if (p.cb) {
      int carry = 0;
      t0 += p.adv_c0;
      if (t0 >= p.cb) {
        t0 -= p.cb;
        carry = 1;
      }
      t1 += p.adv_tap + carry;
      tv += p.adv_tv + carry;
      tu += p.adv_tu;
      if (tv >= p.kw) {
        tv -= p.kw;
        ++tu;
      }
    }
    if (p.kth) {
      int carry = 0;
      kow += p.adv_w * p.wk;
      if (kow >= p.ktw * p.wk) {
        kow -= p.ktw * p.wk;
        carry = 1;
      }
      koh += (p.adv_h + carry) * p.rk;
      carry = 0;
      if (koh >= p.kth * p.rk) {
        koh -= p.kth * p.rk;
        carry = 1;
      }
      kbi += p.adv_b + carry;
    }
  }
  __device__ __forceinline__ void next(const TcArgs& p) {
    ++kb;
    if (p.cb && ++t0 == p.cb) {
      t0 = 0;
      ++t1;
      if (++tv == p.kw) {
        tv = 0;
        ++tu;
      }
    }
    if (p.kth) {
      kow += p.wk;
      if (kow >= p.ktw * p.wk) {
        kow = 0;
        koh += p.rk;
        if (koh >= p.kth * p.rk) {
          koh = 0;
          ++kbi;
        }
      }
    }
  }
};

// Operand loads of one K block, all issued by the producer warp's elected lane; throughput
// comes from several producer warps working on different stages, and boxes stay as large
// as the layout allows (a whole K-major operand tile is one box; MN-major operands are
// 32-float chunks).  Dealing one stage's boxes to several issuers measured slower on
// AlexNet: 2 or 4 lanes of the producer warp -12%, 2 / 3 producer warps -8% / -26%
// (tools/tc_prof.py: the MMA warp waited longer for full stages).
template <int KBLK, bool PAIR>
__device__ __forceinline__ void load_a(const TcArgs& p, const CUtensorMap* map, const Tile& t,
                                       const KCursor& c, int rb, int oh0, int ow0, uint32_t sa,
                                       uint32_t bar) {
  switch (p.a_mode) {
    case A_RECT_K:
      tc::tma_load_4d<PAIR>(sa, map, bar, p.a_c_g * t.g + c.t0 * KBLK, ow0 + p.sign * (c.tv - p.pw),
                            oh0 + p.sign * (c.tu - p.ph), rb);
      break;
    case A_2D_K:
      tc::tma_load_2d<PAIR>(sa, map, bar, c.kb * KBLK, t.m * kTileM);
      break;
    case A_IM2COL_K:
      tc::tma_load_im2col_4d<PAIR>(
          sa, map, bar, p.a_c_g * t.g + c.t0 * KBLK, ow0, oh0, rb,
          static_cast<uint16_t>(p.sign > 0 ? c.tv : p.kw - 1 - c.tv),
          static_cast<uint16_t>(p.sign > 0 ? c.tu : p.kh - 1 - c.tu));
      break;
    case A_RECT_MN:
      for (int j = 0; j < p.a_chunks; ++j)
        tc::tma_load_4d<PAIR>(sa + j * KBLK * 128, map, bar, p.a_c_g * t.g + t.m * kTileM + 32 * j,
                              c.kow, c.koh, c.kbi);
      break;
    case A_2D_MN:
      if (p.a_one) {
        tc::tma_load_3d<PAIR>(sa, map, bar, 0, c.kb * KBLK, (p.a_c_g * t.g + t.m * kTileM) / 32);
        break;
      }
      for (int j = 0; j < p.a_chunks; ++j)
        tc::tma_load_2d<PAIR>(sa + j * KBLK * 128, map, bar, p.a_c_g * t.g + t.m * kTileM + 32 * j,
                              c.kb * KBLK);
      break;
  }
}

template <int KBLK, bool PAIR>
__device__ __forceinline__ void load_b(const TcArgs& p, const CUtensorMap* map,
                                       const CUtensorMap* ones, const Tile& t, const KCursor& c,
                                       int u, int v, const TapChunks& tk, uint32_t sb,
                                       uint32_t bar, int rank) {
  const int nch = (p.b_cols + 31) / 32;
  const int n0 = t.n * p.n_tile + rank * p.b_cols;  // this CTA's first B column
  switch (p.b_mode) {
    case B_2D_K:
      tc::tma_load_2d<PAIR>(sb, map, bar, c.kb * KBLK, p.b_r_g * t.g + n0);
      break;
    case B_WT_MN:  // W viewed as [G][F/G][taps][C/G]: filter blocks past F/G read as 0
      if (p.b_one) {  // [G][taps][C/G / 32][F/G][32]
        tc::tma_load_5d<PAIR>(sb, map, bar, 0, c.t0 * KBLK, n0 / 32, c.t1, t.g);
        break;
      }
      for (int j = 0; j < nch; ++j)
        tc::tma_load_4d<PAIR>(sb + j * KBLK * 128, map, bar, n0 + 32 * j, c.t1, c.t0 * KBLK, t.g);
      break;
    case B_3D_K:  // W viewed as [F][taps][C/G]: channel blocks past C/G read as 0
      tc::tma_load_3d<PAIR>(sb, map, bar, c.t0 * KBLK, c.t1, p.b_r_g * t.g + n0);
      break;
    case B_RECT_MN:
      for (int j = 0; j < nch; ++j)
        tc::tma_load_4d<PAIR>(sb + j * KBLK * 128, map, bar, p.b_n_g * t.g + n0 + 32 * j,
                              c.kow + v - p.pw, c.koh + u - p.ph, c.kbi);
      break;
    case B_2D_MN:
      if (p.b_one) {
        tc::tma_load_3d<PAIR>(sb, map, bar, 0, c.kb * KBLK, n0 / 32);
        break;
      }
      for (int j = 0; j < nch; ++j)
        tc::tma_load_2d<PAIR>(sb + j * KBLK * 128, map, bar, n0 + 32 * j, c.kb * KBLK);
      break;
    case B_COL_MN:  // im2col matrix [G][rows][Kp]: group as the outer coordinate
      for (int j = 0; j < nch; ++j)
        tc::tma_load_3d<PAIR>(sb + j * KBLK * 128, map, bar, n0 + 32 * j, c.kb * KBLK, t.g);
      break;
    case B_TAPS_MN:  // X shifted per 32-column chunk by that chunk's tap
#pragma unroll
      for (int j = 0; j < kMaxBChunks; ++j)
        if (j < nch)
          tc::tma_load_4d<PAIR>(sb + j * KBLK * 128, map, bar, tk.c[j], c.kow + tk.dx[j],
                                c.koh + tk.dy[j], c.kbi);
      break;
    case B_TAPS_IM2COL: {  // the same chunks as TMA im2col boxes over linear pixel K blocks
      const int pix = c.kb * KBLK, r = pix / p.out_w;
      const int x0 = pix - r * p.out_w + p.im_lw, y0 = r % p.out_h + p.im_lh, b0 = r / p.out_h;
#pragma unroll
      for (int j = 0; j < kMaxBChunks; ++j)
        if (j < nch) {
          if (tk.c[j] < 0)  // the bias chunk: a KBLK x 32 box of ones (same bytes)
            tc::tma_load_2d<PAIR>(sb + j * KBLK * 128, ones, bar, 0, 0);
          else
            tc::tma_load_im2col_4d<PAIR>(sb + j * KBLK * 128, map, bar, tk.c[j], x0, y0, b0,
                                         static_cast<uint16_t>(tk.dx[j] + p.pw),
                                         static_cast<uint16_t>(tk.dy[j] + p.ph));
        }
      break;
    }
  }
}

// EPI selects the epilogue features compiled in (each costs registers and time even when
// unused): 0 = fprop (bias / ReLU / split-K partials), 1 = dgrad (+ ReLU mask, accumulate),
// 2 = wgrad (+ multi-tap column map).
template <int KBLK, bool PAIR, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_o, const TcArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], tfull_bar[2], tempty_bar[2];
  __shared__ __align__(16) float bias_sh[2][kAccCols];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // pairs: the cluster is the unit of work; rank 0 (the leader) owns the MMA, the stage
  // "full" barriers (both CTAs' TMA bytes land on them) and the TMEM "empty" barriers
  const int rank = PAIR ? static_cast<int>(tc::cluster_rank()) : 0;
  const long long unit0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const long long ustep = PAIR ? gridDim.x / 2 : gridDim.x;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&map_a);
    tc::tma_prefetch(&map_b);
    if (p.epi_tma || p.bias_chunk) tc::tma_prefetch(&map_o);
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);  // the stage's producer warp, lane 0
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tc::smem_u32(&tfull_bar[b]), 1);
      tc::mbar_init(tc::smem_u32(&tempty_bar[b]), PAIR ? 256 : 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == kAllocWarp) {
    if constexpr (PAIR)
      tc::tmem_alloc_pair(tc::smem_u32(&tmem_base_sh), 2 * kAccCols);
    else
      tc::tmem_alloc(tc::smem_u32(&tmem_base_sh), 2 * kAccCols);
  }
  tc::fence_before_sync();
  if constexpr (PAIR)
    tc::cluster_sync();  // the peer's barriers are initialised before anyone signals them
  else
    __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base_sh;
  pdl_enter();  // setup above touched only smem / TMEM: it overlaps the predecessor's tail

  const int pw = warp < 4 ? warp : (warp == 6 || warp == 7 ? warp - 2 : -1);
  if (pw >= 0 && pw < p.producers && lane == 0) {
    // ----------------------- producers: pipeline stage it (kps K blocks) -> producer it % P
    // Each producer walks only its own stages (the cursor jumps over the others' K blocks),
    // waits for the slot, posts the stage's bytes and issues every box of the stage.
    // pairs: the leader posts both CTAs' bytes (identical per CTA); the peer only loads
    const uint32_t bytes = (p.a_tx + (p.stage_bytes - p.a_bytes)) * (PAIR ? 2 : 1);
    const int P = p.producers;
    const bool prof = p.prof != nullptr && pw == 0 && rank == 0;
    long long prof_t0 = prof ? clock64() : 0, prof_w = 0;
    uint32_t it_tile = 0;  // global stage index of the tile's first stage
    for (long long tt = unit0; tt < p.total_tiles; tt += ustep) {
      Tile t = decode_tile(p, tt);
      if (PAIR) t.m = 2 * t.m + rank;
      const int kb0 = t.split * p.kb_per_split;
      const int kb1 = min(p.kblocks, kb0 + p.kb_per_split);
      const int nst = (kb1 - kb0 + p.kps - 1) / p.kps;
      const int first = static_cast<int>((static_cast<uint32_t>(pw + P) - it_tile % P) % P);
      if (first < nst) {
        int rb = 0, oh0 = 0, ow0 = 0;
        if (p.a_mode == A_RECT_K) {
          rb = t.m / (p.th * p.tw);
          const int r = t.m % (p.th * p.tw);
          oh0 = (r / p.tw) * p.rm;
          ow0 = (r % p.tw) * p.wm;
        } else if (p.a_mode == A_IM2COL_K) {  // the tile's first pixel in traversal coords
          const int pix = t.m * kTileM, r = pix / p.out_w;
          ow0 = pix - r * p.out_w + p.im_lw;
          oh0 = r % p.out_h + p.im_lh;
          rb = r / p.out_h;
        }
        const int u = t.tap / p.kw, v = t.tap % p.kw;
        TapChunks tk;
        if (p.b_mode == B_TAPS_MN || p.b_mode == B_TAPS_IM2COL) tap_chunks(p, t, tk, rank);
        const uint32_t it = it_tile + first;
        uint32_t s = it % p.stages, ph = (it / p.stages) & 1;
        KCursor c;
        c.init(p, kb0 + first * p.kps);
        for (int si = first; si < nst; si += P) {
          const int cnt = min(p.kps, kb1 - (kb0 + si * p.kps));
          const uint32_t bar = PAIR ? tc::mapa(tc::smem_u32(&full_bar[s]), 0)
                                    : tc::smem_u32(&full_bar[s]);
          if (prof) {
            const long long w0 = clock64();
            tc::mbar_wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
            prof_w += clock64() - w0;
          } else {
            tc::mbar_wait(tc::smem_u32(&empty_bar[s]), ph ^ 1);
          }
          if (rank == 0) tc::mbar_arrive_expect_tx(tc::smem_u32(&full_bar[s]), bytes * cnt);
          for (int j = 0; j < cnt; ++j, c.next(p)) {
            const uint32_t sa = tc::smem_u32(smem + (s * p.kps + j) * p.stage_bytes);
            load_a<KBLK, PAIR>(p, &map_a, t, c, rb, oh0, ow0, sa, bar);
            load_b<KBLK, PAIR>(p, &map_b, &map_o, t, c, u, v, tk, sa + p.a_bytes, bar, rank);
          }
          c.advance(p);
          s += P;
          if (s >= static_cast<uint32_t>(p.stages)) {
            s -= p.stages;
            ph ^= 1;
          }
        }
      }
      it_tile += nst;
    }
    if (prof) {
      atomicAdd(p.prof + 4, static_cast<unsigned long long>(prof_w));
      atomicAdd(p.prof + 5, static_cast<unsigned long long>(clock64() - prof_t0));
    }
  } else if (warp == kMmaWarp && rank == 0) {
    // ------------------------------------------------------------ MMA issue
    // The whole warp runs the loop (warp-uniform control flow keeps the descriptors in
    // uniform registers); one elected lane issues.  Descriptors are built once for slot 0
    // and advanced by adding (byte offset >> 4) to the start-address field, so a K block
    // costs a few integer adds per MMA instead of a descriptor build.
    const bool a_mn = p.a_mode == A_RECT_MN || p.a_mode == A_2D_MN;
    const bool b_mn = p.b_mode != B_2D_K && p.b_mode != B_3D_K;
    const uint32_t idesc = tc::idesc_tf32(PAIR ? 2 * kTileM : kTileM, p.n_tile, a_mn, b_mn);
    const uint32_t k_sw = KBLK == 32 ? tc::kSw128 : tc::kSw64;
    const uint32_t k_sbo = 8 * KBLK * 4;  // 8 rows of KBLK floats
    const uint32_t s0 = tc::smem_u32(smem);
    const uint64_t a_desc0 = a_mn ? tc::smem_desc(s0, KBLK * 128, 512, tc::kSw128Base32)
                                  : tc::smem_desc(s0, 16, k_sbo, k_sw);
    const uint64_t b_desc0 = b_mn ? tc::smem_desc(s0 + p.a_bytes, KBLK * 128, 512, tc::kSw128Base32)
                                  : tc::smem_desc(s0 + p.a_bytes, 16, k_sbo, k_sw);
    const uint32_t a_step = (a_mn ? 1024u : 32u) >> 4, b_step = (b_mn ? 1024u : 32u) >> 4;
    const uint32_t slot_step = static_cast<uint32_t>(p.stage_bytes) >> 4;
    const bool leader = tc::elect_one();
    const bool prof = p.prof != nullptr;
    long long prof_t0 = prof ? clock64() : 0, prof_wf = 0, prof_wt = 0, prof_n = 0;
    uint32_t st = 0, ph = 0, local = 0;  // ring slot and its parity
    for (long long tt = unit0; tt < p.total_tiles; tt += ustep, ++local) {
      const Tile t = decode_tile(p, tt);
      const int kb0 = t.split * p.kb_per_split;
      const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
      const uint32_t acc = local & 1;
      if (prof) {
        const long long w0 = clock64();
        tc::mbar_wait(tc::smem_u32(&tempty_bar[acc]), ((local >> 1) & 1) ^ 1);
        prof_wt += clock64() - w0;
      } else {
        tc::mbar_wait(tc::smem_u32(&tempty_bar[acc]), ((local >> 1) & 1) ^ 1);
      }
      tc::fence_after_sync();
      const uint32_t d = tmem + acc * kAccCols;
      for (int i = 0; i < nkb;) {
        const int cnt = min(p.kps, nkb - i);
        const uint32_t s = st;
        if (prof) {
          const long long w0 = clock64();
          tc::mbar_wait(tc::smem_u32(&full_bar[s]), ph);
          prof_wf += clock64() - w0;
          ++prof_n;
        } else {
          tc::mbar_wait(tc::smem_u32(&full_bar[s]), ph);
        }
        tc::fence_after_sync();
        if (leader) {
          uint32_t off = s * static_cast<uint32_t>(p.kps) * slot_step;
          for (int q = 0; q < cnt; ++q, ++i, off += slot_step) {
#pragma unroll
            for (int j = 0; j < KBLK / 8; ++j) {
              const uint64_t ad = a_desc0 + off + j * a_step;
              const uint64_t bd = b_desc0 + off + j * b_step;
              if constexpr (PAIR)
                tc::mma_tf32_pair(d, ad, bd, idesc, (i | j) != 0 ? 1u : 0u);
              else
                tc::mma_tf32(d, ad, bd, idesc, (i | j) != 0 ? 1u : 0u);
            }
          }
          if constexpr (PAIR)
            tc::mma_commit_pair(tc::smem_u32(&empty_bar[s]), 3);
          else
            tc::mma_commit(tc::smem_u32(&empty_bar[s]));
        } else {
          i += cnt;
        }
        __syncwarp();
        if (++st == static_cast<uint32_t>(p.stages)) {
          st = 0;
          ph ^= 1;
        }
      }
      if (leader) {
        if constexpr (PAIR)
          tc::mma_commit_pair(tc::smem_u32(&tfull_bar[acc]), 3);
        else
          tc::mma_commit(tc::smem_u32(&tfull_bar[acc]));
      }
      __syncwarp();
    }
    if (prof && lane == 0) {
      atomicAdd(p.prof + 0, static_cast<unsigned long long>(clock64() - prof_t0));
      atomicAdd(p.prof + 1, static_cast<unsigned long long>(prof_wf));
      atomicAdd(p.prof + 2, static_cast<unsigned long long>(prof_wt));
      atomicAdd(p.prof + 3, static_cast<unsigned long long>(prof_n));
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;
    uint32_t local = 0;
    uint32_t ochunk = 0;  // TMA-store chunks issued by this warp (staging buffer ochunk % 2)
    uint8_t* const ostage = smem + p.ring_bytes + ew * p.epi_tma * kOutChunkBytes;
    const bool prof = p.prof != nullptr && ew == 0 && rank == 0;
    long long prof_t0 = prof ? clock64() : 0, prof_w = 0;
    for (long long tt = unit0; tt < p.total_tiles; tt += ustep, ++local) {
      Tile t = decode_tile(p, tt);
      if (PAIR) t.m = 2 * t.m + rank;
      const int m = ew * 32 + lane;
      bool row_ok;
      long long out_row;
      if (p.row_map == ROW_RECT) {
        const int rb = t.m / (p.th * p.tw);
        const int r = t.m % (p.th * p.tw);
        const int oh = (r / p.tw) * p.rm + m / p.wm, ow = (r % p.tw) * p.wm + m % p.wm;
        row_ok = oh < p.out_h && ow < p.out_w && t.m < p.m_tiles;  // pairs: odd tail tile
        out_row = (static_cast<long long>(rb) * p.out_h + oh) * p.out_w + ow;
      } else {
        const int mm = t.m * kTileM + m;
        row_ok = mm < p.m_valid;
        out_row = static_cast<long long>(p.row_g) * t.g + mm;
      }
      float* base = (p.ws ? p.ws + t.split * p.ws_stride : p.out);
      const long long row_off = out_row * p.ldo;
      const int col0 = p.col_g * t.g + p.col_tap * t.tap + t.n * p.n_tile;
      const int nvalid = min(p.n_tile, p.n_valid - t.n * p.n_tile);
      const uint32_t acc = local & 1;
      // the tile's bias to smem while its MMAs run (safe to overwrite: every epilogue thread
      // passed tile local-1's barrier, so tile local-2's reads of this buffer are done)
      const float* bsh = bias_sh[acc];
      if (p.bias && !p.ws) {
        for (int i = ew * 32 + lane; i < p.n_tile; i += 128)
          bias_sh[acc][i] = i < nvalid ? p.bias[col0 + i] : 0.f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if (prof) {
        const long long w0 = clock64();
        tc::mbar_wait(tc::smem_u32(&tfull_bar[acc]), (local >> 1) & 1);
        prof_w += clock64() - w0;
      } else {
        tc::mbar_wait(tc::smem_u32(&tfull_bar[acc]), (local >> 1) & 1);
      }
      tc::fence_after_sync();
      const uint32_t taddr = tmem + acc * kAccCols + (static_cast<uint32_t>(ew * 32) << 16);
      // Thread = one accumulator row (its TMEM lane): the 32-column chunks stream out of
      // TMEM double-buffered (the load of chunk c0+32 overlaps the stores of chunk c0) and
      // go straight to global memory as float4 runs of the thread's row (no smem
      // transpose); bias / ReLU / accumulate applied in registers.
      const int c_end = __any_sync(0xffffffffu, row_ok) ? p.n_tile : 0;  // idle rows: skip
      const bool tma_rows = p.row_g == 0 || __all_sync(0xffffffffu, row_ok);
      constexpr bool DG = EPI == 1, WG = EPI == 2;
      const bool acc_out = DG && p.accumulate && !p.ws;
      const float* mask = DG ? p.mask : nullptr;
      const int cpt = p.cpt;  // wgrad multi-tap column map (WG only)
      float* rowp = base + row_off;
      uint32_t va[32], vb[32];
      if (c_end > 0) {
        tc::tmem_ld32_async(taddr, va);
        tc::tmem_wait_ld();
      }
      for (int c0 = 0; c0 < c_end; c0 += 32) {
        const bool more = c0 + 32 < c_end;
        if (more) tc::tmem_ld32_async(taddr + c0 + 32, vb);
        // operands the epilogue reads (ReLU mask, accumulated output): all 8 float4 of the
        // chunk are loaded before any store, so the loads overlap instead of each waiting
        // behind the previous store (out / mask may alias as far as the compiler knows)
        float4 pre[8];  // the ReLU mask, else the accumulated output
#ifdef PSG_EPI_NO_PRELOAD
        const bool vec_pre = false;
#else
        const bool vec_pre = DG && row_ok && p.epi_vec && !p.ws;
#endif
        if (vec_pre && (mask || acc_out)) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const int c = c0 + 4 * q4;
            if (c >= nvalid) continue;
            pre[q4] = mask ? __ldg(reinterpret_cast<const float4*>(mask + row_off + col0 + c))
                           : *reinterpret_cast<const float4*>(rowp + col0 + c);
          }
        }
        if (EPI != 2 && p.epi_tma && c0 + 32 <= nvalid && tma_rows) {
          // whole 32-column chunk: registers -> swizzled smem -> one TMA store of the warp's
          // 32 rows (rows past the output / split are clipped by the map's bounds; with
          // per-group row ranges (row_g > 0) only when all 32 rows are the tile's own — a
          // partial chunk would overwrite the next group's rows, which another CTA writes)
          uint8_t* buf = ostage + (p.epi_tma == 2 ? (ochunk & 1) * kOutChunkBytes : 0);
          if (lane == 0) {  // this buffer's previous store has read it
            if (p.epi_tma == 2)
              tc::bulk_wait_read<1>();
            else
              tc::bulk_wait_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const int c = c0 + 4 * q4;
            float4 y = make_float4(__uint_as_float(va[4 * q4]), __uint_as_float(va[4 * q4 + 1]),
                                   __uint_as_float(va[4 * q4 + 2]), __uint_as_float(va[4 * q4 + 3]));
            if (!p.ws) {
              if (p.bias) {
                const float4 bb = *reinterpret_cast<const float4*>(bsh + c);
                y.x += bb.x; y.y += bb.y; y.z += bb.z; y.w += bb.w;
                if (p.relu) {
                  y.x = y.x > 0.f ? y.x : 0.f;
                  y.y = y.y > 0.f ? y.y : 0.f;
                  y.z = y.z > 0.f ? y.z : 0.f;
                  y.w = y.w > 0.f ? y.w : 0.f;
                }
              }
              if (row_ok && mask) {
                const float4 m = vec_pre ? pre[q4]
                                         : *reinterpret_cast<const float4*>(mask + row_off + col0 + c);
                y.x = m.x > 0.f ? y.x : 0.f;
                y.y = m.y > 0.f ? y.y : 0.f;
                y.z = m.z > 0.f ? y.z : 0.f;
                y.w = m.w > 0.f ? y.w : 0.f;
              }
              if (row_ok && acc_out) {
                const float4 o = vec_pre && !mask ? pre[q4]
                                                  : *reinterpret_cast<const float4*>(rowp + col0 + c);
                y.x += o.x; y.y += o.y; y.z += o.z; y.w += o.w;
              }
            }
            *reinterpret_cast<float4*>(buf + lane * 128 + ((q4 ^ (lane & 7)) << 4)) = y;
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int orow = static_cast<int>(out_row - lane);  // the warp's first row
            if (p.ws)
              tc::tma_store_3d(&map_o, tc::smem_u32(buf), col0 + c0, orow, t.split);
            else
              tc::tma_store_2d(&map_o, tc::smem_u32(buf), col0 + c0, orow);
            tc::bulk_commit();
          }
          ++ochunk;
        } else if (row_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const int c = c0 + 4 * q4;  // column within the tile
            int cidx;
            bool ok;
            if (WG && cpt) {
              const int vc = t.n * p.n_tile + c, tap = vc / cpt, cc = vc % cpt;
              ok = c < p.n_tile && tap < p.ntaps && cc < p.cgs;
              cidx = tap * p.cgs + cc;
              if (p.bias_chunk && vc == 32 * p.bias_chunk) {  // every ones column = dbias[f]
                const float bsum = __uint_as_float(va[4 * q4]);
                if (p.ws)
                  p.db_part[static_cast<long long>(t.split) * p.db_ld + out_row] = bsum;
                else
                  p.db[out_row] = bsum;
              }
            } else {
              ok = c < nvalid;
              cidx = col0 + c;
            }
            if (!ok) continue;
            float4 y = make_float4(__uint_as_float(va[4 * q4]), __uint_as_float(va[4 * q4 + 1]),
                                   __uint_as_float(va[4 * q4 + 2]), __uint_as_float(va[4 * q4 + 3]));
            if (p.epi_vec) {
              float4* dst = reinterpret_cast<float4*>(rowp + cidx);
              if (!p.ws) {
                if (p.bias) {
                  const float4 bb = *reinterpret_cast<const float4*>(bsh + c);
                  y.x += bb.x; y.y += bb.y; y.z += bb.z; y.w += bb.w;
                  if (p.relu) {
                    y.x = y.x > 0.f ? y.x : 0.f;
                    y.y = y.y > 0.f ? y.y : 0.f;
                    y.z = y.z > 0.f ? y.z : 0.f;
                    y.w = y.w > 0.f ? y.w : 0.f;
                  }
                }
                if (mask) {
                  const float4 m = vec_pre ? pre[q4]
                                           : *reinterpret_cast<const float4*>(mask + row_off + cidx);
                  y.x = m.x > 0.f ? y.x : 0.f;
                  y.y = m.y > 0.f ? y.y : 0.f;
                  y.z = m.z > 0.f ? y.z : 0.f;
                  y.w = m.w > 0.f ? y.w : 0.f;
                }
                if (acc_out) {
                  const float4 o = vec_pre && !mask ? pre[q4] : *dst;
                  y.x += o.x; y.y += o.y; y.z += o.z; y.w += o.w;
                }
              }
              *dst = y;
            } else {  // unaligned outputs: element stores, each column checked
              const float e4[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                int ce;
                bool oke;
                if (WG && cpt) {
                  const int vc = t.n * p.n_tile + c + e, tap = vc / cpt, cc = vc % cpt;
                  oke = c + e < p.n_tile && tap < p.ntaps && cc < p.cgs;
                  ce = tap * p.cgs + cc;
                } else {
                  oke = c + e < nvalid;
                  ce = col0 + c + e;
                }
                if (!oke) continue;
                float yv = e4[e];
                if (!p.ws) {
                  if (p.bias) {
                    yv += bsh[c + e];
                    if (p.relu) yv = yv > 0.f ? yv : 0.f;
                  }
                  if (mask && !(mask[row_off + ce] > 0.f)) yv = 0.f;
                  if (acc_out) yv += rowp[ce];
                }
                rowp[ce] = yv;
              }
            }
          }
        }
        if (more) {
          tc::tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; ++q) va[q] = vb[q];
        }
      }
      tc::fence_before_sync();
      if constexpr (PAIR)
        tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&tempty_bar[acc]), 0));
      else
        mbar_arrive(tc::smem_u32(&tempty_bar[acc]));
    }
    if (EPI != 2 && p.epi_tma && lane == 0) tc::bulk_wait_all();  // stores done before exit
    if (prof && lane == 0) {
      atomicAdd(p.prof + 6, static_cast<unsigned long long>(prof_w));
      atomicAdd(p.prof + 7, static_cast<unsigned long long>(clock64() - prof_t0));
    }
  }
  tc::fence_before_sync();
  if constexpr (PAIR)
    tc::cluster_sync();  // the peer's remote arrivals / MMA reads of our smem are done
  else
    __syncthreads();
  if (warp == kAllocWarp) {
    tc::fence_after_sync();
    if constexpr (PAIR)
      tc::tmem_dealloc_pair(tmem, 2 * kAccCols);
    else
      tc::tmem_dealloc(tmem, 2 * kAccCols);
  }
}

}  // namespace tck
}  // namespace psg
