// MatMul elementary task on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Used when the three tilers of a `matmul` task are the canonical GEMM triple
// up to leading dimensions / operand majorness:
//     a: off = ca + sa_m*m + sa_k*k     b: off = cb + sb_n*n + sb_k*k
//     c: off = cc + ldc*m + n           repetition space [M, N], pattern [K]
// The launch covers the linear repetition range [first, first+count) of [M, N]
// (one reference launch, refexec.py:488-490); the epilogue masks the ragged
// first/last rows, so unaligned shards (D = 3, 5, ...) are exact.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B k-blocks -> 4-stage smem ring (128B swizzle)
//   warp 1      MMA issuer:   one thread issues tcgen05.mma 128x256x8 into TMEM
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4..7  epilogue:     tcgen05.ld TMEM -> registers -> masked st.global
// Two accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "aol_async.cuh"
#include "aol_common.cuh"

namespace aol {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 32, STAGES = 4;
constexpr int UMMA_K = 8;                       // tf32: 32 bytes of K per MMA
constexpr int A_BYTES = BM * BK * 4;            // 16 KB
constexpr int B_BYTES = BN * BK * 4;            // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KB
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 16;                     // tile raster: 16 M-tiles share each B panel
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
  float* c;            // C + cc
  int64_t ldc;
  int64_t M, N, K;
  int64_t m_lo, m_hi;  // inclusive row range of this launch
  int64_t row_base;    // first row of the tile grid: m_lo, aligned down to 32 rows when A is MN-major
                       // (a TMA box starting off a 128 B swizzle atom faults: illegal instruction)
  int64_t first, last; // inclusive linear repetition range
  int m_tiles, n_tiles, k_blocks, num_tiles;
  int c_vec;           // 16-byte stores allowed
  int group_m;         // tile raster: M-tiles per group sharing each B panel
  int epi_smem;        // pair kernel: stage 32x32 chunks through shared memory for row-contiguous stores
  int chunk_kb;        // 3xtf32: k-blocks accumulated in TMEM between round-to-nearest adds
  int hi_round;        // 3xtf32: 1 = hi rounded to tf32 (rna) and written back; 0 = hi = tensor-core truncation
  // pair kernel, split-K tail: tiles [0, dp_tiles) run whole, one per pair per wave; each of the
  // sk_tiles tail tiles is cut into sk_split k-ranges, and the pieces (k-range major, so the
  // pieces running together read the same k-slices) are dealt to the pairs like tiles.  A
  // tile's partial accumulators are summed in k order by whichever piece arrives last.
  int dp_tiles;
  int sk_tiles, sk_split;
  float* sk_ws;        // [piece][2 CTAs][4 warps][8 chunks][8 col quads][32 lanes][4] fp32 partials
  unsigned* sk_cnt;    // [sk tiles][2 CTAs][4 warps] arrival counters (reset by the last arriver)
  // pair kernel, mixed-width column tiles (w_narrow > 0): each row of m-tiles is cut into
  // n_wide 256-column tiles then n_narrow w_narrow-column tiles, wide tiles dealt first, so
  // every pair gets about the same number of columns (C2's 8-rank shard: 17 x 256 + 20 x 192
  // per row -> 448 columns per pair instead of 2 x 256)
  int n_wide, n_narrow, w_narrow;
};

// ------------------------------------------------------------ PTX helpers ----
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets row (lane base + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor (tcgen05 "version 1").  layout: 2 = SWIZZLE_128B,
// 1 = SWIZZLE_128B_BASE32B (128B swizzle with 32-byte atoms, the only MN-major tf32 layout).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// Operand tile of R rows (M or N) x BK:
//   K-major : one TMA box {BK, R}; rows of 128 B; 8-row atoms 1024 B apart (SBO);
//             the k-th MMA slice starts 32 B further inside the swizzle row.
//   MN-major: R/32 boxes {32, BK} with the 128B/32B-atom swizzle; each box = BK rows
//             (k) of 32 elements (128 B); boxes 4 KB apart (LBO), 4-k-row atoms
//             512 B apart (SBO); the k-th MMA slice starts 8 rows (1024 B) further.
template <bool KMAJOR>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int k) {
  if (KMAJOR) return smem_desc(base + k * (UMMA_K * 4), 16, 1024, 2);
  return smem_desc(base + k * (UMMA_K * 128), BK * 128, 512, 1);
}

template <bool KMAJOR, int R>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, uint64_t* bar, uint8_t* dst, int kcoord,
                                             int rcoord) {
  if (KMAJOR) {
    tma_load_2d(map, bar, dst, kcoord, rcoord);
  } else {
#pragma unroll
    for (int c = 0; c < R / 32; ++c) tma_load_2d(map, bar, dst + c * (BK * 128), rcoord + 32 * c, kcoord);
  }
}

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& mt, int& nt) {
  const int per_group = GROUP_M * p.n_tiles;
  const int g = tile / per_group;
  const int first_m = g * GROUP_M;
  const int gm = min(GROUP_M, p.m_tiles - first_m);
  const int in = tile - g * per_group;
  mt = first_m + in % gm;
  nt = in / gm;
}

template <bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tf32(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer ----
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        int mt, nt;
        tile_coords(p, tile, mt, nt);
        const int row0 = (int)(p.row_base + (int64_t)mt * BM), col0 = nt * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          load_operand<A_KMAJOR, BM>(&map_a, &full[stage], sa, kb * BK, row0);
          load_operand<B_KMAJOR, BN>(&map_b, &full[stage], sb, kb * BK, col0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------ MMA issuer ----
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                 ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k)
            tc_mma_tf32(d_tmem, operand_desc<A_KMAJOR>(sa, k), operand_desc<B_KMAJOR>(sb, k), idesc,
                        (kb | k) != 0);
          tc_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------- epilogue ----
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      int mt, nt;
      tile_coords(p, tile, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t gm = p.row_base + (int64_t)mt * BM + ew * 32 + lane;
      const bool row_ok = gm >= p.m_lo && gm <= p.m_hi && gm < p.M;
      int64_t col_lo = 0, col_hi = p.N;
      if (gm == p.m_lo) col_lo = p.first - p.m_lo * p.N;
      if (gm == p.m_hi) col_hi = p.last - p.m_hi * p.N + 1;
      float* crow = p.c + gm * p.ldc;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + ch * 32, v);
        const int64_t c0 = (int64_t)nt * BN + ch * 32;
        if (!row_ok) continue;
        if (p.c_vec && c0 >= col_lo && c0 + 32 <= col_hi) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(crow + c0 + j) =
                make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                            __uint_as_float(v[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j >= col_lo && c0 + j < col_hi) crow[c0 + j] = __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// =============================================================================
// 2-CTA variant (cta_group::2): a cluster of two CTAs on a TPC computes a 256x256
// tile.  Each CTA TMA-loads its 128 rows of A and its 128 columns of B into its own
// smem (6-stage ring, 32 KB/stage) and signals the leader's full barrier; the
// leader's single thread issues tcgen05.mma.cta_group::2 M=256 N=256, which reads
// both CTAs' operands; each CTA's TMEM holds its 128 rows x 256 fp32 columns.
// Per-SM operand traffic is 2/3 of the 1-CTA 128x256 kernel's.
// =============================================================================
namespace pair {

constexpr int BM = 256, BN = 256, STAGES = 6;
constexpr int HALF_M = 128, HALF_N = 128;
constexpr int A_BYTES = HALF_M * BK * 4;           // 16 KB
constexpr int B_BYTES = HALF_N * BK * 4;           // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;     // 32 KB per CTA
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;        // shared::cluster address of the same offset in CTA 0
constexpr int EPI_PITCH = 33;                     // padded 32x32 staging: conflict-free both ways
constexpr int EPI_BYTES = 4 * 32 * EPI_PITCH * 4;  // one 32x32 fp32 chunk per epilogue warp
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256 + EPI_BYTES;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar, void* dst, int x,
                                                 int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void commit_pair_multicast(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & PEER_MASK) : "memory");
}

template <bool KMAJOR, int R>
__device__ __forceinline__ void load_operand_pair(const CUtensorMap* map, uint32_t leader_bar, uint8_t* dst,
                                                  int kcoord, int rcoord) {
  if (KMAJOR) {
    tma_load_2d_pair(map, leader_bar, dst, kcoord, rcoord);
  } else {
#pragma unroll
    for (int c = 0; c < R / 32; ++c) tma_load_2d_pair(map, leader_bar, dst + c * (BK * 128), rcoord + 32 * c, kcoord);
  }
}

__device__ __forceinline__ void tile_coords_pair(const Params& p, int tile, int& mt, int& nt) {
  const int per_group = p.group_m * p.n_tiles;
  const int g = tile / per_group;
  const int first_m = g * p.group_m;
  const int gm = min(p.group_m, p.m_tiles - first_m);
  const int in = tile - g * per_group;
  mt = first_m + in % gm;
  nt = in / gm;
}

// Output tile `tile` of the pair kernel: its m-tile, first column and width (256, or
// w_narrow for the narrow tiles of a mixed-width plan).
template <bool MIXED>
__device__ __forceinline__ void tile_geom(const Params& p, int tile, int& mt, int& col0, int& width) {
  if (!MIXED) {
    int nt;
    tile_coords_pair(p, tile, mt, nt);
    col0 = nt * BN;
    width = BN;
    return;
  }
  const int wide = p.m_tiles * p.n_wide;
  if (tile < wide) {
    mt = tile % p.m_tiles;
    col0 = (tile / p.m_tiles) * BN;
    width = BN;
  } else {
    const int u = tile - wide;
    mt = u % p.m_tiles;
    col0 = p.n_wide * BN + (u / p.m_tiles) * p.w_narrow;
    width = p.w_narrow;
  }
}

// B operand of one CTA for a tile `width` columns wide (this CTA's half: width / 2 columns
// from rcoord).  MN-major: (width / 2) / 32 boxes of 32 columns; K-major: one box of the
// map's HALF_N rows (rows past the half are loaded and not used).  Returns the bytes issued.
template <bool KMAJOR>
__device__ __forceinline__ uint32_t load_b_pair(const CUtensorMap* map, uint32_t leader_bar, uint8_t* dst, int kcoord,
                                                int rcoord, int half) {
  if (KMAJOR) {
    tma_load_2d_pair(map, leader_bar, dst, kcoord, rcoord);
    return (uint32_t)B_BYTES;
  }
  for (int c = 0; c < half / 32; ++c) tma_load_2d_pair(map, leader_bar, dst + c * (BK * 128), rcoord + 32 * c, kcoord);
  return (uint32_t)(half / 32) * (BK * 128);
}

// One unit of a pair's work: k-blocks [kb0, kb1) of output tile `tile`; `piece` >= 0 for a
// split-K piece of a tail tile (its partial accumulator goes through sk_ws).
struct Unit {
  int tile, kb0, kb1, piece;
};

// Pair `pid` of `np`: whole tiles pid, pid + np, ... below dp_tiles, then tail pieces
// pid, pid + np, ... below sk_tiles * sk_split; piece j is k-range j / sk_tiles of tail tile
// j % sk_tiles.  Every role of the pair (producer, MMA issuer, epilogue) walks the same sequence.
struct UnitIter {
  const Params& p;
  int np, next_tile, next_piece;
  __device__ UnitIter(const Params& p_, int pid, int np_) : p(p_), np(np_), next_tile(pid), next_piece(pid) {}
  __device__ bool next(Unit& u) {
    if (next_tile < p.dp_tiles) {
      u.tile = next_tile;
      u.kb0 = 0;
      u.kb1 = p.k_blocks;
      u.piece = -1;
      next_tile += np;
      return true;
    }
    if (next_piece >= p.sk_tiles * p.sk_split) return false;
    const int kq = next_piece / p.sk_tiles;
    u.tile = p.dp_tiles + (next_piece - kq * p.sk_tiles);
    u.kb0 = (int)((int64_t)p.k_blocks * kq / p.sk_split);
    u.kb1 = (int)((int64_t)p.k_blocks * (kq + 1) / p.sk_split);
    u.piece = next_piece;
    next_piece += np;
    return true;
  }
};

__device__ __forceinline__ float* sk_slot(const Params& p, int piece, uint32_t rank, int ew) {
  return p.sk_ws + (((int64_t)piece * 2 + rank) * 4 + ew) * (int64_t)(8 * 32 * 32);
}

// Masked store of one 32x32 fp32 chunk (rows = the warp's 32 TMEM lanes, columns c0..c0+31)
// into C, staged through padded shared memory so each 16-byte store covers 4 rows x 128 B.
__device__ __forceinline__ void store_chunk(const Params& p, float* epi, int ew, int lane, int mt, int tcol0,
                                            uint32_t rank, int ch, const float (&v)[32]) {
  const int64_t c0 = (int64_t)tcol0 + ch * 32;
  if (p.epi_smem) {
    float* st = epi + ew * 32 * EPI_PITCH;
#pragma unroll
    for (int j = 0; j < 32; ++j) st[lane * EPI_PITCH + j] = v[j];
    __syncwarp();
    const int64_t row0 = p.row_base + (int64_t)mt * BM + rank * HALF_M + ew * 32;
#pragma unroll
    for (int rr = 0; rr < 32; rr += 4) {
      const int r = rr + (lane >> 3), cc = 4 * (lane & 7);
      const int64_t g = row0 + r;
      const float* sp = st + r * EPI_PITCH + cc;
      if (g < p.m_lo || g > p.m_hi || g >= p.M) continue;
      int64_t lo = 0, hi = p.N;
      if (g == p.m_lo) lo = p.first - p.m_lo * p.N;
      if (g == p.m_hi) hi = p.last - p.m_hi * p.N + 1;
      float* dst = p.c + g * p.ldc + c0 + cc;
      const int64_t col = c0 + cc;
      if (p.c_vec && col >= lo && col + 4 <= hi) {
        *reinterpret_cast<float4*>(dst) = make_float4(sp[0], sp[1], sp[2], sp[3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (col + u >= lo && col + u < hi) dst[u] = sp[u];
      }
    }
    __syncwarp();
    return;
  }
  const int64_t gm = p.row_base + (int64_t)mt * BM + rank * HALF_M + ew * 32 + lane;
  if (!(gm >= p.m_lo && gm <= p.m_hi && gm < p.M)) return;
  int64_t col_lo = 0, col_hi = p.N;
  if (gm == p.m_lo) col_lo = p.first - p.m_lo * p.N;
  if (gm == p.m_hi) col_hi = p.last - p.m_hi * p.N + 1;
  float* crow = p.c + gm * p.ldc;
  if (p.c_vec && c0 >= col_lo && c0 + 32 <= col_hi) {
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(crow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c0 + j >= col_lo && c0 + j < col_hi) crow[c0 + j] = v[j];
  }
}

// MIXED: the mixed-width tile plan (run-time tile widths); false compiles the whole-tile
// kernel with every width a constant.
template <bool A_KMAJOR, bool B_KMAJOR, bool MIXED>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tf32_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* epi = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------- TMA producer (both CTAs) ----
      int stage = 0;
      uint32_t phase = 0;
      UnitIter units(p, pair_id, num_pairs);
      Unit u;
      while (units.next(u)) {
        int mt, tcol0, width;
        tile_geom<MIXED>(p, u.tile, mt, tcol0, width);
        const int half = MIXED ? width >> 1 : HALF_N;
        const int row0 = (int)(p.row_base + (int64_t)mt * BM) + (int)rank * HALF_M;
        const int col0 = tcol0 + (int)rank * half;
        const uint32_t b_bytes = (B_KMAJOR || !MIXED) ? (uint32_t)B_BYTES : (uint32_t)(half / 32) * (BK * 128);
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t lbar = smem_u32(&full[stage]) & PEER_MASK;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * ((uint32_t)A_BYTES + b_bytes));
          load_operand_pair<A_KMAJOR, HALF_M>(&map_a, lbar, sa, kb * BK, row0);
          if (MIXED) load_b_pair<B_KMAJOR>(&map_b, lbar, sb, kb * BK, col0, half);
          else load_operand_pair<B_KMAJOR, HALF_N>(&map_b, lbar, sb, kb * BK, col0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------------------------------------------- MMA issuer (leader) ----
      constexpr uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                  ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      UnitIter units(p, pair_id, num_pairs);
      Unit u;
      while (units.next(u)) {
        int mt, tcol0, width;
        tile_geom<MIXED>(p, u.tile, mt, tcol0, width);
        const uint32_t idesc = idesc0 | ((uint32_t)((MIXED ? width : BN) >> 3) << 17);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k)
            mma_tf32_pair(d_tmem, operand_desc<A_KMAJOR>(sa, k), operand_desc<B_KMAJOR>(sb, k), idesc,
                          (kb != u.kb0 || k != 0) ? 1u : 0u);
          commit_pair_multicast(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        commit_pair_multicast(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------- epilogue (both CTAs) ----
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    UnitIter units(p, pair_id, num_pairs);
    Unit u;
    while (units.next(u)) {
      int mt, tcol0, width;
      tile_geom<MIXED>(p, u.tile, mt, tcol0, width);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      if (u.piece < 0) {
        const int nch = MIXED ? width / 32 : BN / 32;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          store_chunk(p, epi, ew, lane, mt, tcol0, rank, ch, v);
        }
        tc_fence_before();
        arrive_leader(&tempty[acc]);
      } else {
        // split-K piece: park the partial accumulator (coalesced [chunk][col][lane]), free the
        // TMEM buffer, then count arrivals; the last piece sums all of them in k order
        float* mine = sk_slot(p, u.piece, rank, ew);
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          float4* dst = reinterpret_cast<float4*>(mine) + ch * 8 * 32 + lane;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4)
            __stcg(dst + j4 * 32, make_float4(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]),
                                              __uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])));
        }
        tc_fence_before();
        arrive_leader(&tempty[acc]);
        const int t_sk = u.tile - p.dp_tiles;
        unsigned* cnt = p.sk_cnt + ((int64_t)t_sk * 2 + rank) * 4 + ew;
        __threadfence();
        __syncwarp();
        unsigned prev = 0;
        if (lane == 0) prev = atomicAdd(cnt, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == (unsigned)(p.sk_split - 1)) {
          __threadfence();
#pragma unroll 1
          for (int ch = 0; ch < BN / 32; ++ch) {
            // partials in k order; two pieces' loads in flight per round (16 x 16 B per lane)
            float v[32];
            const float4* s0 = reinterpret_cast<const float4*>(sk_slot(p, t_sk, rank, ew)) + ch * 8 * 32 + lane;
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 a = __ldcg(s0 + j4 * 32);
              v[4 * j4] = a.x; v[4 * j4 + 1] = a.y; v[4 * j4 + 2] = a.z; v[4 * j4 + 3] = a.w;
            }
            int kq = 1;
            for (; kq + 1 < p.sk_split; kq += 2) {
              const float4* s1 = reinterpret_cast<const float4*>(sk_slot(p, kq * p.sk_tiles + t_sk, rank, ew)) +
                                 ch * 8 * 32 + lane;
              const float4* s2 = reinterpret_cast<const float4*>(
                                     sk_slot(p, (kq + 1) * p.sk_tiles + t_sk, rank, ew)) + ch * 8 * 32 + lane;
              float4 b1[8], b2[8];
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                b1[j4] = __ldcg(s1 + j4 * 32);
                b2[j4] = __ldcg(s2 + j4 * 32);
              }
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                v[4 * j4] += b1[j4].x; v[4 * j4 + 1] += b1[j4].y; v[4 * j4 + 2] += b1[j4].z; v[4 * j4 + 3] += b1[j4].w;
              }
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                v[4 * j4] += b2[j4].x; v[4 * j4 + 1] += b2[j4].y; v[4 * j4 + 2] += b2[j4].z; v[4 * j4 + 3] += b2[j4].w;
              }
            }
            if (kq < p.sk_split) {
              const float4* s1 = reinterpret_cast<const float4*>(sk_slot(p, kq * p.sk_tiles + t_sk, rank, ew)) +
                                 ch * 8 * 32 + lane;
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 b = __ldcg(s1 + j4 * 32);
                v[4 * j4] += b.x; v[4 * j4 + 1] += b.y; v[4 * j4 + 2] += b.z; v[4 * j4 + 3] += b.w;
              }
            }
            store_chunk(p, epi, ew, lane, mt, tcol0, rank, ch, v);
          }
          if (lane == 0) *cnt = 0u;             // ready for the next launch on this scratch
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace pair

// =============================================================================
// fp32-faithful MatMul (precision="3xtf32"), fused: C = Alo.B + A.Blo + A.B with
// A = Ahi + Alo, B = Bhi + Blo (hi = x truncated to tf32, lo = x - hi exactly), all three
// products on the tensor cores from ONE fp32 TMA load of each operand tile.
//   warp 0      TMA producer (each CTA): fp32 A 128x32 and B 64x32 k-blocks -> its own
//               smem ring, completion on its own full barrier
//   warps 8-11  converters (each CTA): write lo = x - hi next to the landed tile, where hi is
//               x with its 13 low mantissa bits dropped -- exactly what kind::tf32 reads
//               from an fp32 container (measured: TF32-level error otherwise), so the tile
//               itself is the hi operand; fence.proxy.async, arrive on the leader's conv
//               barrier.  (AOL_3XTF32_HI=1: hi rounded to nearest and written back instead.)
//   warp 1      MMA issuer (leader CTA): per k-slice tcgen05.mma cta_group::2 kind::tf32
//               M=256 N=128 for lo.hi, hi.lo then hi.hi
//   warps 4-7   epilogue (each CTA): the tensor core's fp32 accumulation rounds toward
//               zero, so its error grows linearly with K (3xtf32 through one accumulator:
//               1.9e-5 normwise at K = 8192); here TMEM accumulates K-chunks of 64 only
//               (two accumulators, alternating) and the epilogue adds each chunk into a
//               running sum R in TMEM with round-to-nearest fp32 adds (tcgen05.ld/st),
//               storing R after the last chunk.
// TMEM: acc0 cols 0-127, acc1 cols 128-255, R cols 256-383.
// =============================================================================
namespace x3 {

constexpr int BM = 256, BN = 128, HALF_M = 128, HALF_N = 64, STAGES = 4, CHUNK_KB = 2;
constexpr int NUM_THREADS = 384;
constexpr int A_BYTES = HALF_M * BK * 4;              // 16 KB fp32 (rewritten as hi)
constexpr int B_BYTES = HALF_N * BK * 4;              // 8 KB
constexpr int LO_OFF = A_BYTES + B_BYTES;             // lo copies follow, same layout
constexpr int STAGE_BYTES = 2 * LO_OFF;               // 48 KB per CTA
constexpr int R_COL = 256;
constexpr int EPI_PITCH = 33;
constexpr int EPI_BYTES = 4 * 32 * EPI_PITCH * 4;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256 + EPI_BYTES;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <bool KMAJOR, int R>
__device__ __forceinline__ void load_operand_local(const CUtensorMap* map, uint64_t* bar, uint8_t* dst, int kcoord,
                                                   int rcoord) {
  if (KMAJOR) {
    tma_load_2d(map, bar, dst, kcoord, rcoord);
  } else {
#pragma unroll
    for (int c = 0; c < R / 32; ++c) tma_load_2d(map, bar, dst + c * (BK * 128), rcoord + 32 * c, kcoord);
  }
}

template <bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_3xtf32_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       Params p) {
  using pair::arrive_leader;
  using pair::cluster_rank;
  using pair::cluster_sync;
  using pair::commit_pair_multicast;
  using pair::mma_tf32_pair;
  using pair::PEER_MASK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;
  uint64_t* tfull = conv + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* epi = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
  const int chunk_kb = p.chunk_kb;
  const int n_chunks = (p.k_blocks + chunk_kb - 1) / chunk_kb;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 2 * 128);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------- TMA producer (both CTAs) ----
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        int mt, nt;
        pair::tile_coords_pair(p, tile, mt, nt);
        const int row0 = (int)(p.row_base + (int64_t)mt * BM) + (int)rank * HALF_M;
        const int col0 = nt * BN + (int)rank * HALF_N;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          load_operand_local<A_KMAJOR, HALF_M>(&map_a, &full[stage], sa, kb * BK, row0);
          load_operand_local<B_KMAJOR, HALF_N>(&map_b, &full[stage], sa + A_BYTES, kb * BK, col0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------ converters (both CTAs) ----
    const int t = threadIdx.x - 256;
    const uint32_t cbar0 = smem_u32(&conv[0]) & PEER_MASK;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        float4* x = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES);
        float4* lo = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES + LO_OFF);
        if (p.hi_round) {
#pragma unroll
          for (int i = t; i < LO_OFF / 16; i += 128) {
            const float4 v = x[i];
            float4 h, l;
            h.x = tf32_rna(v.x); l.x = __fsub_rn(v.x, h.x);
            h.y = tf32_rna(v.y); l.y = __fsub_rn(v.y, h.y);
            h.z = tf32_rna(v.z); l.z = __fsub_rn(v.z, h.z);
            h.w = tf32_rna(v.w); l.w = __fsub_rn(v.w, h.w);
            x[i] = h;
            lo[i] = l;
          }
        } else {
          // hi = x with the 13 low mantissa bits dropped, which is what the tensor core
          // reads from an fp32 container; only lo is written
#pragma unroll
          for (int i = t; i < LO_OFF / 16; i += 128) {
            const float4 v = x[i];
            float4 l;
            l.x = __fsub_rn(v.x, __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
            l.y = __fsub_rn(v.y, __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
            l.z = __fsub_rn(v.z, __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
            l.w = __fsub_rn(v.w, __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
            lo[i] = l;
          }
        }
        fence_proxy_async_smem();            // generic-proxy writes -> visible to the tensor core
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cbar0 + stage * 8) : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------------------------------------------- MMA issuer (leader) ----
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                 ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        for (int c = 0; c < n_chunks; ++c) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          const int kb_end = min(p.k_blocks, (c + 1) * chunk_kb);
          for (int kb = c * chunk_kb; kb < kb_end; ++kb) {
            mbar_wait(&conv[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t ah = operand_desc<A_KMAJOR>(sa, k), al = operand_desc<A_KMAJOR>(sa + LO_OFF, k);
              const uint64_t bh = operand_desc<B_KMAJOR>(sb, k), bl = operand_desc<B_KMAJOR>(sb + LO_OFF, k);
              mma_tf32_pair(d_tmem, al, bh, idesc, (kb != c * chunk_kb) || (k != 0));
              mma_tf32_pair(d_tmem, ah, bl, idesc, 1u);
              mma_tf32_pair(d_tmem, ah, bh, idesc, 1u);
            }
            commit_pair_multicast(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          commit_pair_multicast(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------- epilogue (both CTAs) ----
    const int ew = warp - 4;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
      int mt, nt;
      pair::tile_coords_pair(p, tile, mt, nt);
      for (int c = 0; c < n_chunks; ++c) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const bool last = (c == n_chunks - 1);
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t v[32];
          tmem_ld32(tmem_base + lane_base + acc * BN + ch * 32, v);
          if (c > 0) {
            uint32_t r[32];
            tmem_ld32(tmem_base + lane_base + R_COL + ch * 32, r);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              v[j] = __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __uint_as_float(v[j])));
          }
          if (!last) {
            tmem_st32(tmem_base + lane_base + R_COL + ch * 32, v);
            continue;
          }
          // final chunk: transpose the 32x32 block through padded smem, row-contiguous stores
          const int64_t c0 = (int64_t)nt * BN + ch * 32;
          float* st = epi + ew * 32 * EPI_PITCH;
#pragma unroll
          for (int j = 0; j < 32; ++j) st[lane * EPI_PITCH + j] = __uint_as_float(v[j]);
          __syncwarp();
          const int64_t row0 = p.row_base + (int64_t)mt * BM + rank * HALF_M + ew * 32;
#pragma unroll
          for (int rr = 0; rr < 32; rr += 4) {
            const int r = rr + (lane >> 3), cc = 4 * (lane & 7);
            const int64_t g = row0 + r;
            const float* sp = st + r * EPI_PITCH + cc;
            if (g < p.m_lo || g > p.m_hi || g >= p.M) continue;
            int64_t lo = 0, hi = p.N;
            if (g == p.m_lo) lo = p.first - p.m_lo * p.N;
            if (g == p.m_hi) hi = p.last - p.m_hi * p.N + 1;
            float* dst = p.c + g * p.ldc + c0 + cc;
            const int64_t col = c0 + cc;
            if (p.c_vec && col >= lo && col + 4 <= hi) {
              *reinterpret_cast<float4*>(dst) = make_float4(sp[0], sp[1], sp[2], sp[3]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (col + u >= lo && col + u < hi) dst[u] = sp[u];
            }
          }
          __syncwarp();
        }
        if (!last) tmem_wait_st();
        tc_fence_before();
        arrive_leader(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace x3

// =============================================================================
// 3xTF32, wide form (default): the same three products as x3 above on a 256x256 pair tile
// (M=256 N=256 per tcgen05.mma, the shape the TF32 kernel runs at), A and B hi/lo in shared
// memory.  TMEM cannot hold two 256-column chunk accumulators AND the running sum, so the
// accumulator is single: cols 0-255 accumulate one K chunk, cols 256-511 hold R.  Sixteen
// epilogue warps (four per TMEM lane quarter, 64 columns each) fold a finished chunk into R
// with round-to-nearest adds and release the accumulator; the MMA issuer waits for that
// release before the next chunk, so the fold is kept short (two 32-column pieces per warp).
// Same chunking and add order as x3: bit-identical results.
//   warp 0 TMA producer, warp 1 MMA issuer (leader), warp 2 TMEM allocator,
//   warps 4-7 and 12-23 epilogue, warps 8-11 converters.  3 stages x 64 KB per CTA.
// =============================================================================
namespace x3w {

constexpr int BM = 256, BN = 256, HALF_M = 128, HALF_N = 128, STAGES = 3, CHUNK_KB = 2;
constexpr int NUM_THREADS = 768, EPI_THREADS = 512;
constexpr int A_BYTES = HALF_M * BK * 4;              // 16 KB
constexpr int B_BYTES = HALF_N * BK * 4;              // 16 KB
constexpr int LO_OFF = A_BYTES + B_BYTES;             // lo copies follow, same layout
constexpr int STAGE_BYTES = 2 * LO_OFF;               // 64 KB per CTA
constexpr int R_COL = 256;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;

template <bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_3xtf32_wide(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       Params p) {
  using pair::arrive_leader;
  using pair::cluster_rank;
  using pair::cluster_sync;
  using pair::commit_pair_multicast;
  using pair::mma_tf32_pair;
  using pair::PEER_MASK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;
  uint64_t* tfull = conv + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
  const int chunk_kb = p.chunk_kb;
  const int n_chunks = (p.k_blocks + chunk_kb - 1) / chunk_kb;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 2 * 128);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * EPI_THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------- TMA producer (both CTAs) ----
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        int mt, nt;
        pair::tile_coords_pair(p, tile, mt, nt);
        const int row0 = (int)(p.row_base + (int64_t)mt * BM) + (int)rank * HALF_M;
        const int col0 = nt * BN + (int)rank * HALF_N;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          x3::load_operand_local<A_KMAJOR, HALF_M>(&map_a, &full[stage], sa, kb * BK, row0);
          x3::load_operand_local<B_KMAJOR, HALF_N>(&map_b, &full[stage], sa + A_BYTES, kb * BK, col0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ------------------------------------------------------ converters (both CTAs) ----
    const int t = threadIdx.x - 256;
    const uint32_t cbar0 = smem_u32(&conv[0]) & PEER_MASK;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        float4* x = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES);
        float4* lo = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES + LO_OFF);
        if (p.hi_round) {
#pragma unroll 4
          for (int i = t; i < LO_OFF / 16; i += 128) {
            const float4 v = x[i];
            float4 h, l;
            h.x = x3::tf32_rna(v.x); l.x = __fsub_rn(v.x, h.x);
            h.y = x3::tf32_rna(v.y); l.y = __fsub_rn(v.y, h.y);
            h.z = x3::tf32_rna(v.z); l.z = __fsub_rn(v.z, h.z);
            h.w = x3::tf32_rna(v.w); l.w = __fsub_rn(v.w, h.w);
            x[i] = h;
            lo[i] = l;
          }
        } else {
#pragma unroll 4
          for (int i = t; i < LO_OFF / 16; i += 128) {
            const float4 v = x[i];
            float4 l;
            l.x = __fsub_rn(v.x, __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
            l.y = __fsub_rn(v.y, __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
            l.z = __fsub_rn(v.z, __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
            l.w = __fsub_rn(v.w, __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
            lo[i] = l;
          }
        }
        x3::fence_proxy_async_smem();
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cbar0 + stage * 8) : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------------------------------------------- MMA issuer (leader) ----
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                 ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        for (int c = 0; c < n_chunks; ++c) {
          mbar_wait(tempty, acc_phase ^ 1);            // the epilogue has folded the previous chunk
          tc_fence_after();
          const int kb_end = min(p.k_blocks, (c + 1) * chunk_kb);
          for (int kb = c * chunk_kb; kb < kb_end; ++kb) {
            mbar_wait(&conv[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t ah = operand_desc<A_KMAJOR>(sa, k), al = operand_desc<A_KMAJOR>(sa + LO_OFF, k);
              const uint64_t bh = operand_desc<B_KMAJOR>(sb, k), bl = operand_desc<B_KMAJOR>(sb + LO_OFF, k);
              mma_tf32_pair(tmem_base, al, bh, idesc, (kb != c * chunk_kb) || (k != 0));
              mma_tf32_pair(tmem_base, ah, bl, idesc, 1u);
              mma_tf32_pair(tmem_base, ah, bh, idesc, 1u);
            }
            commit_pair_multicast(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          commit_pair_multicast(tfull);
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------- epilogue (both CTAs, warps 4-7 and 12-23) ----
    const int q = warp & 3;                              // TMEM lane quarter (warp id mod 4)
    const int slice = warp < 8 ? 0 : (warp - 8) >> 2;    // columns slice*64 .. +63
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t acc_phase = 0;
    for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
      int mt, nt;
      pair::tile_coords_pair(p, tile, mt, nt);
      const int64_t g = p.row_base + (int64_t)mt * BM + rank * HALF_M + q * 32 + lane;
      const bool row_ok = g >= p.m_lo && g <= p.m_hi && g < p.M;
      int64_t lo_col = 0, hi_col = p.N;
      if (g == p.m_lo) lo_col = p.first - p.m_lo * p.N;
      if (g == p.m_hi) hi_col = p.last - p.m_hi * p.N + 1;
      for (int c = 0; c < n_chunks; ++c) {
        mbar_wait(tfull, acc_phase);
        acc_phase ^= 1;
        tc_fence_after();
        const bool last = (c == n_chunks - 1);
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const uint32_t col = (uint32_t)(slice * 64 + ch * 32);
          uint32_t v[32];
          tmem_ld32(tmem_base + lane_base + col, v);
          if (c > 0) {
            uint32_t r[32];
            tmem_ld32(tmem_base + lane_base + R_COL + col, r);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              v[j] = __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __uint_as_float(v[j])));
          }
          if (!last) {
            x3::tmem_st32(tmem_base + lane_base + R_COL + col, v);
            continue;
          }
          // final chunk: this thread's row, 32 consecutive columns, straight to C
          if (!row_ok) continue;
          const int64_t c0 = (int64_t)nt * BN + col;
          float* dst = p.c + g * p.ldc + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const int64_t cc = c0 + j;
            if (p.c_vec && cc >= lo_col && cc + 4 <= hi_col) {
              *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                                __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (cc + u >= lo_col && cc + u < hi_col) dst[j + u] = __uint_as_float(v[j + u]);
            }
          }
        }
        if (!last) x3::tmem_wait_st();
        tc_fence_before();
        arrive_leader(tempty);
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace x3w

// =============================================================================
// 3xTF32, register form: the wide kernel's 256x256 pair tiles and shared-memory operands, but
// the running sum R lives in registers, so TMEM holds TWO 256-column chunk accumulators
// (cols 0-255, 256-511) and the MMAs never wait for a fold.  Ten warps (320 threads, so a
// thread may hold 204 registers): warp 0 TMA producer + TMEM allocator, warp 1 MMA issuer,
// warps 2-9 both convert (lo = x - hi next to each landed tile) and fold: warp w owns TMEM
// lane quarter w % 4 and columns ((w - 2) / 4) * 128 .. +127, i.e. 128 fp32 of R per thread.
// They walk the chunks of their tiles in order: convert chunk j's k-blocks, then fold chunk
// j - 1 (its accumulator is full by then: the MMAs of chunk j still have work converted), so
// the fold overlaps the tensor cores.  Same chunks and add order as x3 / x3w: same bits.
// =============================================================================
namespace x3r {

constexpr int BM = 256, BN = 256, HALF_M = 128, HALF_N = 128, STAGES = 3, CHUNK_KB = 2;
constexpr int NUM_THREADS = 320, WORK_THREADS = 256;
constexpr int A_BYTES = HALF_M * BK * 4;              // 16 KB
constexpr int B_BYTES = HALF_N * BK * 4;              // 16 KB
constexpr int LO_OFF = A_BYTES + B_BYTES;
constexpr int STAGE_BYTES = 2 * LO_OFF;               // 64 KB per CTA
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;

template <bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_3xtf32_regs(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       Params p) {
  using pair::arrive_leader;
  using pair::cluster_rank;
  using pair::cluster_sync;
  using pair::commit_pair_multicast;
  using pair::mma_tf32_pair;
  using pair::PEER_MASK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;
  uint64_t* tfull = conv + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
  const int chunk_kb = p.chunk_kb;
  const int n_chunks = (p.k_blocks + chunk_kb - 1) / chunk_kb;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 2 * WORK_THREADS);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * WORK_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------- TMA producer (both CTAs) ----
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        int mt, nt;
        pair::tile_coords_pair(p, tile, mt, nt);
        const int row0 = (int)(p.row_base + (int64_t)mt * BM) + (int)rank * HALF_M;
        const int col0 = nt * BN + (int)rank * HALF_N;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          x3::load_operand_local<A_KMAJOR, HALF_M>(&map_a, &full[stage], sa, kb * BK, row0);
          x3::load_operand_local<B_KMAJOR, HALF_N>(&map_b, &full[stage], sa + A_BYTES, kb * BK, col0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------------------------------------------- MMA issuer (leader) ----
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_KMAJOR ? 0u : 1u) << 15) |
                                 ((B_KMAJOR ? 0u : 1u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
        for (int c = 0; c < n_chunks; ++c) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);      // this accumulator's previous chunk was read
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          const int kb_end = min(p.k_blocks, (c + 1) * chunk_kb);
          for (int kb = c * chunk_kb; kb < kb_end; ++kb) {
            mbar_wait(&conv[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t ah = operand_desc<A_KMAJOR>(sa, k), al = operand_desc<A_KMAJOR>(sa + LO_OFF, k);
              const uint64_t bh = operand_desc<B_KMAJOR>(sb, k), bl = operand_desc<B_KMAJOR>(sb + LO_OFF, k);
              mma_tf32_pair(d_tmem, al, bh, idesc, (kb != c * chunk_kb) || (k != 0));
              mma_tf32_pair(d_tmem, ah, bl, idesc, 1u);
              mma_tf32_pair(d_tmem, ah, bh, idesc, 1u);
            }
            commit_pair_multicast(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          commit_pair_multicast(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------ converters + folds (both CTAs, warps 2-9) ----
    const int t = threadIdx.x - 64;
    const int q = warp & 3;                              // TMEM lane quarter
    const int half = (warp - 2) >> 2;                    // columns half*128 .. +127
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t cbar0 = smem_u32(&conv[0]) & PEER_MASK;
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    float R[4][32];
    // fold chunk `c` of tile (fmt, fnt) from accumulator `acc` into R; store R after its last chunk
    auto fold = [&](int c, int fmt, int fnt) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
        tmem_ld32(tmem_base + lane_base + acc * BN + half * 128 + ch * 32, v);
        if (c == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) R[ch][j] = __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) R[ch][j] = __fadd_rn(R[ch][j], __uint_as_float(v[j]));
        }
      }
      tc_fence_before();
      arrive_leader(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (c != n_chunks - 1) return;
      const int64_t g = p.row_base + (int64_t)fmt * BM + rank * HALF_M + q * 32 + lane;
      if (g < p.m_lo || g > p.m_hi || g >= p.M) return;
      int64_t lo_col = 0, hi_col = p.N;
      if (g == p.m_lo) lo_col = p.first - p.m_lo * p.N;
      if (g == p.m_hi) hi_col = p.last - p.m_hi * p.N + 1;
      const int64_t c0 = (int64_t)fnt * BN + half * 128;
      float* dst = p.c + g * p.ldc + c0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int64_t cc = c0 + ch * 32 + j;
          if (p.c_vec && cc >= lo_col && cc + 4 <= hi_col) {
            *reinterpret_cast<float4*>(dst + ch * 32 + j) =
                make_float4(R[ch][j], R[ch][j + 1], R[ch][j + 2], R[ch][j + 3]);
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (cc + u >= lo_col && cc + u < hi_col) dst[ch * 32 + j + u] = R[ch][j + u];
          }
        }
      }
    };
    int pc = -1, pmt = 0, pnt = 0;                       // the chunk waiting to be folded
    for (int tile = pair_id; tile < p.num_tiles; tile += num_pairs) {
      int mt, nt;
      pair::tile_coords_pair(p, tile, mt, nt);
      for (int c = 0; c < n_chunks; ++c) {
        const int kb_end = min(p.k_blocks, (c + 1) * chunk_kb);
        for (int kb = c * chunk_kb; kb < kb_end; ++kb) {
          mbar_wait(&full[stage], phase);
          float4* x = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES);
          float4* lo = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES + LO_OFF);
          if (p.hi_round) {
#pragma unroll 2
            for (int i = t; i < LO_OFF / 16; i += WORK_THREADS) {
              const float4 v = x[i];
              float4 h, l;
              h.x = x3::tf32_rna(v.x); l.x = __fsub_rn(v.x, h.x);
              h.y = x3::tf32_rna(v.y); l.y = __fsub_rn(v.y, h.y);
              h.z = x3::tf32_rna(v.z); l.z = __fsub_rn(v.z, h.z);
              h.w = x3::tf32_rna(v.w); l.w = __fsub_rn(v.w, h.w);
              x[i] = h;
              lo[i] = l;
            }
          } else {
#pragma unroll 2
            for (int i = t; i < LO_OFF / 16; i += WORK_THREADS) {
              const float4 v = x[i];
              float4 l;
              l.x = __fsub_rn(v.x, __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
              l.y = __fsub_rn(v.y, __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
              l.z = __fsub_rn(v.z, __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
              l.w = __fsub_rn(v.w, __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
              lo[i] = l;
            }
          }
          x3::fence_proxy_async_smem();
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cbar0 + stage * 8) : "memory");
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (pc >= 0) fold(pc, pmt, pnt);
        pc = c; pmt = mt; pnt = nt;
      }
    }
    if (pc >= 0) fold(pc, pmt, pnt);
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace x3r

// ------------------------------------------------------------ host side ----

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace gemm

void* tensor_map_encoder() { return reinterpret_cast<void*>(gemm::encode_fn()); }

namespace gemm {

// 2-D fp32 tensor map: dims {inner, outer}, row pitch in elements, box {bi, bo}, 128B swizzle.
static int make_map(CUtensorMap* map, const float* base, int64_t inner, int64_t outer, int64_t pitch, int bi,
                    int bo, bool kmajor) {
  auto fn = encode_fn();
  if (!fn) return fail(AOL_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(pitch * 4)};
  cuuint32_t box[2] = {(cuuint32_t)bi, (cuuint32_t)bo};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  kmajor ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(AOL_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return AOL_OK;
}

}  // namespace gemm

// Canonical-GEMM recognition from the affine forms of the three tilers.
struct GemmShape {
  bool ok;
  bool a_kmajor, b_kmajor;
  int64_t M, N, K;
  int64_t ca, lda, cb, ldb, cc, ldc;
};

GemmShape recognise_gemm(const aol_task& t) {
  GemmShape g{};
  const aol_tiler &ta = t.tilers[0], &tb = t.tilers[1], &tc = t.tilers[2];
  if (ta.rep_rank != 2 || tb.rep_rank != 2 || tc.rep_rank != 2) return g;
  if (tiler_pat_total(ta) != ta.pattern[ta.pat_rank - 1]) return g;  // pattern must be 1-D (after extent-1 dims)
  if (tiler_pat_total(tb) != tb.pattern[tb.pat_rank - 1]) return g;
  Affine a = tiler_affine(ta), b = tiler_affine(tb), c = tiler_affine(tc);
  if (!a.ok || !b.ok || !c.ok) return g;
  const int64_t M = ta.rep[0], N = ta.rep[1], K = tiler_pat_total(ta);
  const int64_t sa_m = a.A[0], sa_n = a.A[1], sa_k = a.B[ta.pat_rank - 1];
  const int64_t sb_m = b.A[0], sb_n = b.A[1], sb_k = b.B[tb.pat_rank - 1];
  if (sa_n != 0 || sb_m != 0) return g;                      // a depends on m only, b on n only
  if (c.A[1] != 1 || c.A[0] < N) return g;                   // c row-major with ldc >= N
  bool ak = (sa_k == 1 && sa_m >= K), am = (sa_m == 1 && sa_k >= M);
  bool bn = (sb_n == 1 && sb_k >= N), bk = (sb_k == 1 && sb_n >= K);
  if (!(ak || am) || !(bn || bk)) return g;
  g.a_kmajor = ak;
  g.b_kmajor = bk && !bn;
  g.lda = ak ? sa_m : sa_k;
  g.ldb = g.b_kmajor ? sb_n : sb_k;
  g.M = M; g.N = N; g.K = K;
  g.ca = a.c0; g.cb = b.c0; g.cc = c.c0; g.ldc = c.A[0];
  // TMA: 16-byte aligned bases and pitches, coordinates inside int32
  if ((g.lda % 4) || (g.ldb % 4) || (g.ca % 4) || (g.cb % 4)) return g;
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31)) return g;
  g.ok = true;
  return g;
}

bool gemm_tf32_applicable(const aol_task& t, void* const* ports) {
  if (t.dtype != AOL_F32) return false;
  if (t.precision == AOL_PREC_EXACT) return false;
  GemmShape g = recognise_gemm(t);
  if (!g.ok) return false;
  const float* a = static_cast<const float*>(ports[0]) + g.ca;
  const float* b = static_cast<const float*>(ports[1]) + g.cb;
  return ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0);
}

int launch_gemm_tf32(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t stream);

// Exact-order MatMul (precision="exact", or dtypes / alignments the tensor-core path does not
// take) for canonical GEMM tilers with any strides: a 64x64 output tile per 256-thread CTA, 4x4
// outputs per thread, K staged through shared memory 16 at a time.  Every output accumulates
// k = 0, 1, ... with the product and the sum rounded separately (__fmul_rn then __fadd_rn, no
// FMA) -- the reference spmv order the oracle pins -- so results are bit-identical to the
// one-thread-per-repetition kernel, at CUDA-core throughput instead of a strided K loop.
struct GemmStrides {
  int64_t M, N, K, ca, sam, sak, cb, sbk, sbn, cc, scm, scn;
};

bool recognise_gemm_strides(const aol_task& t, GemmStrides& g) {
  const aol_tiler &ta = t.tilers[0], &tb = t.tilers[1], &tc = t.tilers[2];
  if (ta.rep_rank != 2 || tb.rep_rank != 2 || tc.rep_rank != 2) return false;
  if (tiler_pat_total(ta) != ta.pattern[ta.pat_rank - 1] || tiler_pat_total(tb) != tb.pattern[tb.pat_rank - 1])
    return false;
  Affine a = tiler_affine(ta), b = tiler_affine(tb), c = tiler_affine(tc);
  if (!a.ok || !b.ok || !c.ok) return false;
  if (a.A[1] != 0 || b.A[0] != 0) return false;          // a depends on m only, b on n only
  g.M = ta.rep[0]; g.N = ta.rep[1]; g.K = tiler_pat_total(ta);
  g.ca = a.c0; g.sam = a.A[0]; g.sak = a.B[ta.pat_rank - 1];
  g.cb = b.c0; g.sbk = b.B[tb.pat_rank - 1]; g.sbn = b.A[1];
  g.cc = c.c0; g.scm = c.A[0]; g.scn = c.A[1];
  return g.M < (1ll << 31) && g.N < (1ll << 31);
}

bool recognise_gemm_strides(const aol_task& t) {
  GemmStrides g;
  return recognise_gemm_strides(t, g);
}

constexpr int EX_T = 64, EX_K = 16;

template <typename T>
__device__ __forceinline__ T ex_mac(T acc, T a, T b);
template <> __device__ __forceinline__ float ex_mac(float acc, float a, float b) { return __fadd_rn(acc, __fmul_rn(a, b)); }
template <> __device__ __forceinline__ double ex_mac(double acc, double a, double b) { return __dadd_rn(acc, __dmul_rn(a, b)); }

template <typename T>
__global__ void __launch_bounds__(256) k_gemm_exact(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                                                    GemmStrides g, int64_t m_lo, int64_t first, int64_t last,
                                                    int n_tiles) {
  __shared__ T As[EX_K][EX_T + 1];
  __shared__ T Bs[EX_K][EX_T + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t mt = blockIdx.x / n_tiles, nt = blockIdx.x - mt * n_tiles;
  const int64_t m0 = m_lo + mt * EX_T, n0 = nt * EX_T;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  for (int64_t k0 = 0; k0 < g.K; k0 += EX_K) {
    // stage a 64 x 16 slab of A and a 16 x 64 slab of B (zero-padded past the edges: the padded
    // products are never added to a stored output's chain)
    for (int e = threadIdx.x; e < EX_T * EX_K; e += 256) {
      const int r = e / EX_K, kk = e % EX_K;
      const int64_t m = m0 + r, k = k0 + kk;
      As[kk][r] = (m < g.M && k < g.K) ? A[g.ca + g.sam * m + g.sak * k] : T(0);
      const int cidx = e % EX_T, kb = e / EX_T;
      const int64_t n = n0 + cidx, k2 = k0 + kb;
      Bs[kb][cidx] = (n < g.N && k2 < g.K) ? B[g.cb + g.sbk * k2 + g.sbn * n] : T(0);
    }
    __syncthreads();
    const int kn = (int)(g.K - k0 < EX_K ? g.K - k0 : EX_K);
    for (int kk = 0; kk < kn; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = ex_mac(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      const int64_t lin = m * g.N + n;
      if (n < g.N && lin >= first && lin <= last) C[g.cc + g.scm * m + g.scn * n] = acc[i][j];
    }
  }
}

// 128 x 128 output tile per CTA (256 threads, 8 x 8 outputs each: rows ty*4 + {0..3} and
// 64 + ty*4 + {0..3}, columns likewise), K through a double-buffered shared-memory slab 8 deep;
// the next slab's global loads are issued before the current slab's products.  Each output
// still accumulates k ascending with a separate rounding per product and per add: the same
// bits as k_gemm_exact (and the oracle).  4x fewer shared-memory operand loads per product
// than the 4 x 4 form, which was bound by them.
constexpr int EX2_T = 128, EX2_K = 8;

template <typename T>
__device__ __forceinline__ void ex_ld4(const T* p, T (&v)[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
    const double2 q0 = reinterpret_cast<const double2*>(p)[0], q1 = reinterpret_cast<const double2*>(p)[1];
    v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_gemm_exact128(const T* __restrict__ A, const T* __restrict__ B,
                                                       T* __restrict__ C, GemmStrides g, int64_t m_lo, int64_t first,
                                                       int64_t last, int n_tiles) {
  __shared__ __align__(16) T As[2][EX2_K][EX2_T];
  __shared__ __align__(16) T Bs[2][EX2_K][EX2_T];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t mt = blockIdx.x / n_tiles, nt = blockIdx.x - mt * n_tiles;
  const int64_t m0 = m_lo + mt * EX2_T, n0 = nt * EX2_T;
  const bool a_k_fast = g.sak == 1, b_n_fast = g.sbn == 1;
  T ra[4], rb[4];
  // slab element e = threadIdx.x + 256 u (u < 4) -> (row/col, k) with the unit-stride axis fastest
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int r = a_k_fast ? e >> 3 : e & 127, kk = a_k_fast ? e & 7 : e >> 7;
      const int64_t m = m0 + r, k = k0 + kk;
      ra[u] = (m < g.M && k < g.K) ? A[g.ca + g.sam * m + g.sak * k] : T(0);
      const int c = b_n_fast ? e & 127 : e >> 3, kb = b_n_fast ? e >> 7 : e & 7;
      const int64_t n = n0 + c, k2 = k0 + kb;
      rb[u] = (n < g.N && k2 < g.K) ? B[g.cb + g.sbk * k2 + g.sbn * n] : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u;
      As[buf][a_k_fast ? e & 7 : e >> 7][a_k_fast ? e >> 3 : e & 127] = ra[u];
      Bs[buf][b_n_fast ? e >> 7 : e & 7][b_n_fast ? e & 127 : e >> 3] = rb[u];
    }
  };
  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < g.K; k0 += EX2_K) {
    const bool more = k0 + EX2_K < g.K;
    if (more) load(k0 + EX2_K);
    const int kn = (int)(g.K - k0 < EX2_K ? g.K - k0 : EX2_K);
    for (int kk = 0; kk < kn; ++kk) {
      T a[8], b[8];
      ex_ld4(&As[buf][kk][ty * 4], *reinterpret_cast<T(*)[4]>(a));
      ex_ld4(&As[buf][kk][64 + ty * 4], *reinterpret_cast<T(*)[4]>(a + 4));
      ex_ld4(&Bs[buf][kk][tx * 4], *reinterpret_cast<T(*)[4]>(b));
      ex_ld4(&Bs[buf][kk][64 + tx * 4], *reinterpret_cast<T(*)[4]>(b + 4));
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = ex_mac(acc[i][j], a[i], b[j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      const int64_t lin = m * g.N + n;
      if (n < g.N && lin >= first && lin <= last) C[g.cc + g.scm * m + g.scn * n] = acc[i][j];
    }
  }
}

int launch_gemm_exact(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t stream) {
  GemmStrides g;
  if (!recognise_gemm_strides(t, g)) return AOL_EUNSUPPORTED;
  if (count <= 0) return AOL_OK;
  const int64_t last = first + count - 1;
  const int64_t m_lo = first / g.N, m_hi = last / g.N;
  // 128 x 128 tiles once there is one per SM (the double-buffered 8 x 8-per-thread form); small
  // products keep 64 x 64 tiles for more CTAs.  AOL_GEMM_EXACT64=1 forces the 64 x 64 form.
  static const bool force64 = getenv("AOL_GEMM_EXACT64") != nullptr;
  const int64_t m_big = (m_hi - m_lo + EX2_T) / EX2_T, n_big = (g.N + EX2_T - 1) / EX2_T;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!force64 && m_big * n_big >= sms && m_big * n_big < (1ll << 31)) {
    const unsigned grid = (unsigned)(m_big * n_big);
    if (t.dtype == AOL_F32)
      k_gemm_exact128<float><<<grid, 256, 0, stream>>>((const float*)ports[0], (const float*)ports[1],
                                                        (float*)ports[2], g, m_lo, first, last, (int)n_big);
    else
      k_gemm_exact128<double><<<grid, 256, 0, stream>>>((const double*)ports[0], (const double*)ports[1],
                                                         (double*)ports[2], g, m_lo, first, last, (int)n_big);
    AOL_LAUNCH_CHECK("k_gemm_exact128");
    return AOL_OK;
  }
  const int64_t m_tiles = (m_hi - m_lo + EX_T) / EX_T, n_tiles = (g.N + EX_T - 1) / EX_T;
  if (m_tiles * n_tiles >= (1ll << 31)) return AOL_EUNSUPPORTED;
  const unsigned grid = (unsigned)(m_tiles * n_tiles);
  if (t.dtype == AOL_F32)
    k_gemm_exact<float><<<grid, 256, 0, stream>>>((const float*)ports[0], (const float*)ports[1], (float*)ports[2], g,
                                                   m_lo, first, last, (int)n_tiles);
  else
    k_gemm_exact<double><<<grid, 256, 0, stream>>>((const double*)ports[0], (const double*)ports[1],
                                                    (double*)ports[2], g, m_lo, first, last, (int)n_tiles);
  AOL_LAUNCH_CHECK("k_gemm_exact");
  return AOL_OK;
}

// Batched MatMul: a repetition space [B..., M, N] whose last two axes form a canonical GEMM for
// every leading index (e.g. a[b, m, k], b[b, k, n], c[b, m, n]).  Each batch slice is the same
// task with a 2-D repetition space [M, N] and the origins advanced by the leading paving
// columns; slices run as ordinary tcgen05 launches over their share of [first, first+count).
static bool gemm_slice(const aol_task& t, int64_t batch, aol_task& out) {
  out = t;
  const int q = t.tilers[0].rep_rank;
  for (int i = 0; i < 3; ++i) {
    const aol_tiler& src = t.tilers[i];
    aol_tiler& dst = out.tilers[i];
    if (src.rep_rank != q) return false;
    // unravel the leading repetition index (row-major over the q-2 leading axes)
    int64_t lead[AOL_MAX_RANK];
    int64_t rem = batch;
    for (int j = q - 3; j >= 0; --j) {
      lead[j] = rem % src.rep[j];
      rem /= src.rep[j];
    }
    dst.rep_rank = 2;
    dst.rep[0] = src.rep[q - 2];
    dst.rep[1] = src.rep[q - 1];
    for (int j = 2; j < AOL_MAX_RANK; ++j) dst.rep[j] = 0;
    for (int d = 0; d < src.arr_rank; ++d) {
      int64_t o = src.origin[d];
      for (int j = 0; j < q - 2; ++j) o += src.paving[d][j] * lead[j];
      dst.origin[d] = o;
      dst.paving[d][0] = src.paving[d][q - 2];
      dst.paving[d][1] = src.paving[d][q - 1];
      for (int j = 2; j < AOL_MAX_RANK; ++j) dst.paving[d][j] = 0;
    }
  }
  return true;
}

bool gemm_batched_applicable(const aol_task& t, void* const* ports) {
  if (t.dtype != AOL_F32 || t.precision == AOL_PREC_EXACT) return false;
  const int q = t.tilers[0].rep_rank;
  if (q < 3 || t.tilers[1].rep_rank != q || t.tilers[2].rep_rank != q) return false;
  int64_t nb = 1;
  for (int j = 0; j < q - 2; ++j) nb *= t.tilers[0].rep[j];
  // every slice must be a TMA-compatible GEMM; checking the first and the last suffices for
  // affine tilers (the origin moves linearly, the strides do not change)
  aol_task s0, s1;
  if (!gemm_slice(t, 0, s0) || !gemm_slice(t, nb - 1, s1)) return false;
  return gemm_tf32_applicable(s0, ports) && gemm_tf32_applicable(s1, ports);
}

int launch_gemm_batched(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t stream) {
  const int q = t.tilers[0].rep_rank;
  const int64_t MN = t.tilers[0].rep[q - 2] * t.tilers[0].rep[q - 1];
  for (int64_t b = first / MN; b * MN < first + count; ++b) {
    const int64_t lo = std::max<int64_t>(first, b * MN), hi = std::min<int64_t>(first + count, (b + 1) * MN);
    aol_task sl;
    if (!gemm_slice(t, b, sl)) return fail(AOL_EINVAL, "batched matmul slice");
    const int rc = launch_gemm_tf32(sl, lo - b * MN, hi - lo, ports, stream);
    if (rc) return rc;
  }
  return AOL_OK;
}

// Batched exact-order MatMul (precision="exact", repetition space [B..., M, N]): every slice
// through the tiled exact kernel, bit-identical to the one-thread-per-repetition kernel (both
// accumulate k = 0, 1, ... with the product and the sum rounded separately).  Returns
// AOL_EUNSUPPORTED (nothing launched) when a slice is not a canonical GEMM.
int launch_gemm_exact_batched(const aol_task& t, int64_t first, int64_t count, void* const* ports,
                              cudaStream_t stream) {
  const int q = t.tilers[0].rep_rank;
  if (q < 3 || t.tilers[1].rep_rank != q || t.tilers[2].rep_rank != q) return AOL_EUNSUPPORTED;
  int64_t nb = 1;
  for (int j = 0; j < q - 2; ++j) nb *= t.tilers[0].rep[j];
  aol_task s0, s1;
  GemmStrides g0, g1;
  if (!gemm_slice(t, 0, s0) || !gemm_slice(t, nb - 1, s1) || !recognise_gemm_strides(s0, g0) ||
      !recognise_gemm_strides(s1, g1))
    return AOL_EUNSUPPORTED;
  const int64_t MN = t.tilers[0].rep[q - 2] * t.tilers[0].rep[q - 1];
  for (int64_t b = first / MN; b * MN < first + count; ++b) {
    const int64_t lo = std::max<int64_t>(first, b * MN), hi = std::min<int64_t>(first + count, (b + 1) * MN);
    aol_task sl;
    if (!gemm_slice(t, b, sl)) return fail(AOL_EINVAL, "batched matmul slice");
    const int rc = launch_gemm_exact(sl, lo - b * MN, hi - lo, ports, stream);
    if (rc) return rc;
  }
  return AOL_OK;
}

bool gemm_exact_batched_applicable(const aol_task& t) {
  const int q = t.tilers[0].rep_rank;
  if (q < 3 || t.tilers[1].rep_rank != q || t.tilers[2].rep_rank != q) return false;
  int64_t nb = 1;
  for (int j = 0; j < q - 2; ++j) nb *= t.tilers[0].rep[j];
  aol_task s0, s1;
  GemmStrides g0, g1;
  return gemm_slice(t, 0, s0) && gemm_slice(t, nb - 1, s1) && recognise_gemm_strides(s0, g0) &&
         recognise_gemm_strides(s1, g1);
}

// Split x into tf32 hi (low 13 mantissa bits cleared) and lo = x - hi (exact).
__global__ void __launch_bounds__(256) k_split_a(const float* __restrict__ A, float* __restrict__ Ap, int64_t rows,
                                                 int64_t K, int64_t sm, int64_t sk, int64_t row0, int64_t pitch) {
  // Ap = [Alo | Ahi | Ahi], row-major [rows, 3K]: the small correction products accumulate
  // first, so they are not rounded away against the large Ahi.Bhi running sum
  const int64_t n = rows * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / K, k = e - r * K;
    const float x = A[(row0 + r) * sm + k * sk];
    const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    const float lo = __fsub_rn(x, hi);
    float* row = Ap + r * pitch;
    row[k] = lo;
    row[K + k] = hi;
    row[2 * K + k] = hi;
  }
}

__global__ void __launch_bounds__(256) k_split_b(const float* __restrict__ B, float* __restrict__ Bp, int64_t K,
                                                 int64_t N, int64_t sk, int64_t sn, int64_t pitch) {
  // Bp = [Bhi ; Blo ; Bhi], row-major [3K, N]
  const int64_t n = K * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / N, c = e - k * N;
    const float x = B[k * sk + c * sn];
    const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    Bp[k * pitch + c] = hi;
    Bp[(K + k) * pitch + c] = __fsub_rn(x, hi);
    Bp[(2 * K + k) * pitch + c] = hi;
  }
}

static int gemm_core(const float* A, const float* B, float* C, const GemmShape& g, int64_t first, int64_t count,
                     cudaStream_t stream);
static int gemm_core_3x(const float* A, const float* B, float* C, const GemmShape& g, int64_t first, int64_t count,
                        cudaStream_t stream);

// Split-K tail scratch per (device, stream): the partial accumulators of the tail pieces and
// the arrival counters of the tail tiles.  Launches on one stream are ordered, launches on
// different streams never share it.  The counters are zeroed once and reset by each tail
// tile's last piece; the partial buffer grows to the largest tail seen.  Bounded like the dot
// scratch; aol_release_scratch() frees it.
struct GemmScratch {
  float* ws = nullptr;
  size_t ws_bytes = 0;
  unsigned* cnt = nullptr;
  uint64_t used = 0;
};
constexpr size_t kMaxGemmScratch = 16;
constexpr int kSkMaxTiles = 1024;
constexpr size_t kSkPieceBytes = (size_t)2 * 4 * 8 * 32 * 32 * sizeof(float);   // 256 KB per piece
static std::mutex g_gemm_mu;
static std::map<std::pair<int, cudaStream_t>, GemmScratch> g_gemm_scratch;
static uint64_t g_gemm_tick = 0;

static void free_gemm_entry(int dev, GemmScratch& e) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  cudaDeviceSynchronize();                        // no kernel still uses it
  cudaFree(e.ws);
  cudaFree(e.cnt);
  cudaSetDevice(cur);
}

static bool gemm_scratch(int dev, cudaStream_t stream, int pieces, float** ws, unsigned** cnt) {
  std::lock_guard<std::mutex> lock(g_gemm_mu);
  auto it = g_gemm_scratch.find({dev, stream});
  if (it == g_gemm_scratch.end()) {
    if (g_gemm_scratch.size() >= kMaxGemmScratch) {
      auto victim = g_gemm_scratch.begin();
      for (auto v = g_gemm_scratch.begin(); v != g_gemm_scratch.end(); ++v)
        if (v->second.used < victim->second.used) victim = v;
      free_gemm_entry(victim->first.first, victim->second);
      g_gemm_scratch.erase(victim);
    }
    GemmScratch e;
    const size_t cnt_bytes = (size_t)kSkMaxTiles * 2 * 4 * sizeof(unsigned);
    if (cudaMalloc(&e.cnt, cnt_bytes) != cudaSuccess) return false;
    if (cudaMemset(e.cnt, 0, cnt_bytes) != cudaSuccess) {
      cudaFree(e.cnt);
      return false;
    }
    it = g_gemm_scratch.emplace(std::make_pair(dev, stream), e).first;
  }
  GemmScratch& e = it->second;
  const size_t need = (size_t)pieces * kSkPieceBytes;
  if (e.ws_bytes < need) {
    if (e.ws) {
      cudaStreamSynchronize(stream);              // the previous launch on this stream is done with it
      cudaFree(e.ws);
      e.ws = nullptr;
      e.ws_bytes = 0;
    }
    if (cudaMalloc(&e.ws, need) != cudaSuccess) return false;
    e.ws_bytes = need;
  }
  e.used = ++g_gemm_tick;
  *ws = e.ws;
  *cnt = e.cnt;
  return true;
}

int release_gemm_scratch() {
  std::lock_guard<std::mutex> lock(g_gemm_mu);
  for (auto& kv : g_gemm_scratch) free_gemm_entry(kv.first.first, kv.second);
  g_gemm_scratch.clear();
  return 0;
}

// Split-K tail of the pair kernel.  Whole waves of tiles run data-parallel.  A last partial
// wave of R = tiles % pairs tiles that would leave pairs idle is cut into s = 2 k-ranges
// (pieces of >= 32 k-blocks) when that shortens it: ceil(2R / pairs) / 2 waves instead of 1
// (R <= pairs / 2; R = 34 of 74, the 4-rank C2 shard: 0.5 waves).  AOL_GEMM_SPLIT=s forces
// s (diagnostics, tests).  Returns s (1 = no split).
static int split_k_tail(int num_tiles, int k_blocks, int pairs) {
  const char* env = getenv("AOL_GEMM_STREAMK");       // read per launch (A/B probes toggle it)
  if (env && env[0] == '0') return 1;
  const int rem = num_tiles % pairs;
  if (rem == 0 || rem > kSkMaxTiles) return 1;
  const char* force = getenv("AOL_GEMM_SPLIT");           // diagnostic: force s (2..8)
  if (force && atoi(force) >= 2 && k_blocks / atoi(force) >= 4) return atoi(force);
  int best = 1;
  double best_t = 1.0;
  // s = 2 only: at more pieces per tile the pieces' epilogues (partial stores, the k-ordered
  // sum) outweigh the shorter tail (tools/time_streamk.py, forced s: 8-rank shard s = 2/3/4/8
  // 0.95/0.93/0.96/0.88x, 4-rank shard s = 3/4/8 0.91/1.03/1.01x; s = 2 at the 4-rank shard
  // 1.09-1.135x)
  for (int sp : {2}) {
    if (k_blocks / sp < 32) break;
    const double t = (double)((rem * sp + pairs - 1) / pairs) / sp;
    if (t < best_t - 1e-9) {
      best_t = t;
      best = sp;
    }
  }
  return best_t <= 0.9 ? best : 1;
}

// Mixed-width column tiles for the pair kernel: when whole 256-column tiles leave the last
// wave partly idle, cut each row of m-tiles into n_wide 256-column tiles then n_narrow tiles
// of w_narrow (192 or 128) columns, with the wide tiles dealt first (tile t to pair t mod
// pairs), if that shortens the busiest pair by >= 4% (opt-in, see below).  A narrow tile still loads the whole A
// block per k-step, so it costs more than its share of columns: measured at 8192^3 with every
// tile w wide (tools/gpu/r2_ncol.sh, AOL_GEMM_NARROW_ALL): 192 -> 0.83x, 128 -> 0.64x,
// 64 -> 0.39x the 256-wide throughput per column, i.e. a 192 / 128 tile takes 0.90 / 0.78 of a
// 256 tile's time.  C2's 8-rank shard (4 rows, 74 pairs): 17 x 256 + 20 x 192 per row, busiest
// pair 1.90 instead of 2 tile times (measured 1.02x); tiny products (one 256 x 256 tile) run
// as two 128-column tiles on two pairs.  Returns false (keep whole tiles) otherwise.
static bool narrow_plan(int m_tiles, int64_t N, int pairs, int& n_wide, int& n_narrow, int& w_narrow) {
  // opt-in (AOL_GEMM_NARROW=1, read per launch): the run-time-width kernel this needs runs
  // 15-20% slower per tile than the constant-width one (same-box A/B: the 8-rank shard 0.31 ms
  // mixed vs 0.25-0.28 ms whole tiles), more than the 5% the plan saves
  const char* env = getenv("AOL_GEMM_NARROW");
  const char* fw = getenv("AOL_GEMM_NARROW_ALL");         // diagnostic: every tile w columns wide
  if (!(env && env[0] == '1') && !fw) return false;
  if (fw && (atoi(fw) == 64 || atoi(fw) == 128 || atoi(fw) == 192)) {
    n_wide = 0;
    w_narrow = atoi(fw);
    n_narrow = (int)((N + w_narrow - 1) / w_narrow);
    return true;
  }
  const int64_t n_full = (N + 255) / 256;
  const int64_t tiles0 = (int64_t)m_tiles * n_full;
  const double base = (double)((tiles0 + pairs - 1) / pairs);  // busiest pair, in 256-tile times
  double best = base;
  bool found = false;
  for (int wn : {192, 128}) {
    const double cost = wn == 192 ? 0.90 : 0.78;           // time of one narrow tile / a 256 tile
    for (int64_t nw = 0; nw * 256 <= N; ++nw) {
      const int64_t nn = (N - nw * 256 + wn - 1) / wn;
      const int64_t wide = (int64_t)m_tiles * nw, total = wide + (int64_t)m_tiles * nn;
      if (total > (int64_t)1 << 30) continue;
      // pair q owns tiles q, q + pairs, ...: ceil((wide - q) / pairs) wide ones, the rest narrow
      double worst = 0.0;
      for (int q = 0; q < pairs && q < total; ++q) {
        const int64_t mine = (total - q + pairs - 1) / pairs;
        const int64_t w = wide > q ? (wide - q + pairs - 1) / pairs : 0;
        worst = std::max(worst, (double)w + (double)(mine - w) * cost);
      }
      if (worst <= base * 0.96 && worst < best - 1e-9) {
        best = worst;
        n_wide = (int)nw;
        n_narrow = (int)nn;
        w_narrow = wn;
        found = true;
      }
    }
  }
  return found;
}

int launch_gemm_tf32(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t stream) {
  GemmShape g = recognise_gemm(t);
  if (!g.ok) return fail(AOL_EUNSUPPORTED, "matmul tilers are not a TMA-compatible GEMM");
  if (count <= 0) return AOL_OK;
  const float* A = static_cast<const float*>(ports[0]) + g.ca;
  const float* B = static_cast<const float*>(ports[1]) + g.cb;
  float* C = static_cast<float*>(ports[2]) + g.cc;
  if (t.precision != AOL_PREC_3XTF32) return gemm_core(A, B, C, g, first, count, stream);
  const char* split_env = getenv("AOL_3XTF32_SPLIT");
  const bool split = split_env != nullptr && split_env[0] == '1';
  if (!split) return gemm_core_3x(A, B, C, g, first, count, stream);
  // diagnostic form (AOL_3XTF32_SPLIT=1): C = Alo.Bhi + Ahi.Blo + Ahi.Bhi as ONE tensor-core
  // GEMM over K' = 3K of K-concatenated operands [Alo|Ahi|Ahi] . [Bhi;Blo;Bhi] materialised in
  // HBM (one fp32 accumulation in TMEM over all of K')
  const int64_t m_lo = first / g.N, m_hi = (first + count - 1) / g.N, rows = m_hi - m_lo + 1;
  const int64_t lda3 = (3 * g.K + 3) / 4 * 4, ldb3 = (g.N + 3) / 4 * 4;   // 16-byte TMA pitches
  float *Ap = nullptr, *Bp = nullptr;
  AOL_CUDA_CHECK(cudaMallocAsync((void**)&Ap, (size_t)rows * lda3 * sizeof(float), stream));
  AOL_CUDA_CHECK(cudaMallocAsync((void**)&Bp, (size_t)3 * g.K * ldb3 * sizeof(float), stream));
  const int64_t sa_m = g.a_kmajor ? g.lda : 1, sa_k = g.a_kmajor ? 1 : g.lda;
  const int64_t sb_k = g.b_kmajor ? 1 : g.ldb, sb_n = g.b_kmajor ? g.ldb : 1;
  k_split_a<<<grid_for(rows * g.K, 256, 16), 256, 0, stream>>>(A, Ap, rows, g.K, sa_m, sa_k, m_lo, lda3);
  AOL_LAUNCH_CHECK("k_split_a");
  k_split_b<<<grid_for(g.K * g.N, 256, 16), 256, 0, stream>>>(B, Bp, g.K, g.N, sb_k, sb_n, ldb3);
  AOL_LAUNCH_CHECK("k_split_b");
  GemmShape g3 = g;
  g3.a_kmajor = true;
  g3.b_kmajor = false;
  g3.M = rows;
  g3.K = 3 * g.K;
  g3.lda = lda3;
  g3.ldb = ldb3;
  int rc = gemm_core(Ap, Bp, C + m_lo * g.ldc, g3, first - m_lo * g.N, count, stream);
  cudaFreeAsync(Ap, stream);
  cudaFreeAsync(Bp, stream);
  return rc;
}

static int gemm_core(const float* A, const float* B, float* C, const GemmShape& g, int64_t first, int64_t count,
                     cudaStream_t stream) {
  using namespace gemm;
  CUtensorMap ma, mb;
  int rc;
  if (g.a_kmajor) rc = make_map(&ma, A, g.K, g.M, g.lda, BK, BM, true);
  else rc = make_map(&ma, A, g.M, g.K, g.lda, 32, BK, false);
  if (rc) return rc;
  if (g.b_kmajor) rc = make_map(&mb, B, g.K, g.N, g.ldb, BK, BN, true);
  else rc = make_map(&mb, B, g.N, g.K, g.ldb, 32, BK, false);
  if (rc) return rc;

  Params p{};
  p.c = C;
  p.ldc = g.ldc;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.first = first;
  p.last = first + count - 1;
  p.m_lo = first / g.N;
  p.m_hi = p.last / g.N;
  p.row_base = g.a_kmajor ? p.m_lo : (p.m_lo & ~int64_t(31));
  p.m_tiles = (int)((p.m_hi - p.row_base + BM) / BM);
  p.n_tiles = (int)((g.N + BN - 1) / BN);
  p.k_blocks = (int)((g.K + BK - 1) / BK);
  p.num_tiles = p.m_tiles * p.n_tiles;
  p.c_vec = ((uintptr_t)C % 16 == 0) && (g.ldc % 4 == 0);

  static const bool force_1sm = getenv("AOL_GEMM_1SM") != nullptr;
  if (!force_1sm) {
    // 2-CTA path: re-encode B with 128-column boxes (each CTA loads half the tile's N)
    CUtensorMap mb2;
    if (g.b_kmajor) rc = make_map(&mb2, B, g.K, g.N, g.ldb, BK, pair::HALF_N, true);
    else rc = make_map(&mb2, B, g.N, g.K, g.ldb, 32, BK, false);
    if (rc) return rc;
    CUtensorMap ma2;
    if (g.a_kmajor) rc = make_map(&ma2, A, g.K, g.M, g.lda, BK, pair::HALF_M, true);
    else rc = make_map(&ma2, A, g.M, g.K, g.lda, 32, BK, false);
    if (rc) return rc;
    Params pp = p;
    static const int gm_env = getenv("AOL_GEMM_GROUP_M") ? atoi(getenv("AOL_GEMM_GROUP_M")) : 0;
    pp.group_m = gm_env > 0 ? gm_env : 8;
    static const char* epi_env = getenv("AOL_GEMM_EPI_SMEM");
    pp.epi_smem = epi_env ? (epi_env[0] != '0') : 1;
    pp.m_tiles = (int)((p.m_hi - p.row_base + pair::BM) / pair::BM);
    pp.n_tiles = (int)((g.N + pair::BN - 1) / pair::BN);
    pp.num_tiles = pp.m_tiles * pp.n_tiles;
    int sms2 = kNumSMs;
    int dev2 = 0;
    if (cudaGetDevice(&dev2) == cudaSuccess) cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev2);
    int pairs = pp.num_tiles < sms2 / 2 ? pp.num_tiles : sms2 / 2;
    pp.dp_tiles = pp.num_tiles;
    pp.sk_tiles = 0;
    pp.sk_split = 1;
    {
      const int all = sms2 / 2;
      const int sp = split_k_tail(pp.num_tiles, pp.k_blocks, all);
      const int rem = pp.num_tiles % all;
      float* ws = nullptr;
      unsigned* cnt = nullptr;
      if (sp > 1 && gemm_scratch(dev2, stream, rem * sp, &ws, &cnt)) {
        pp.dp_tiles = pp.num_tiles - rem;
        pp.sk_tiles = rem;
        pp.sk_split = sp;
        pp.sk_ws = ws;
        pp.sk_cnt = cnt;
        pairs = all;                                   // the pieces spread over every pair
      } else if (narrow_plan(pp.m_tiles, g.N, all, pp.n_wide, pp.n_narrow, pp.w_narrow)) {
        pp.num_tiles = pp.m_tiles * (pp.n_wide + pp.n_narrow);
        pp.dp_tiles = pp.num_tiles;
        pairs = std::min(all, pp.num_tiles);
      }
    }
    void (*k2)(const CUtensorMap, const CUtensorMap, Params);
    const bool mixed = pp.w_narrow != 0;
    if (mixed) {
      if (g.a_kmajor) k2 = g.b_kmajor ? pair::k_gemm_tf32_pair<true, true, true> : pair::k_gemm_tf32_pair<true, false, true>;
      else k2 = g.b_kmajor ? pair::k_gemm_tf32_pair<false, true, true> : pair::k_gemm_tf32_pair<false, false, true>;
    } else {
      if (g.a_kmajor) k2 = g.b_kmajor ? pair::k_gemm_tf32_pair<true, true, false> : pair::k_gemm_tf32_pair<true, false, false>;
      else k2 = g.b_kmajor ? pair::k_gemm_tf32_pair<false, true, false> : pair::k_gemm_tf32_pair<false, false, false>;
    }
    AOL_CUDA_CHECK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair::SMEM_BYTES));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = pair::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    AOL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k2, ma2, mb2, pp));
    AOL_LAUNCH_CHECK("k_gemm_tf32_pair");
    return AOL_OK;
  }
  void (*kern)(const CUtensorMap, const CUtensorMap, Params);
  if (g.a_kmajor) kern = g.b_kmajor ? k_gemm_tf32<true, true> : k_gemm_tf32<true, false>;
  else kern = g.b_kmajor ? k_gemm_tf32<false, true> : k_gemm_tf32<false, false>;
  AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  int sms = kNumSMs;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = p.num_tiles < sms ? p.num_tiles : sms;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ma, mb, p);
  AOL_LAUNCH_CHECK("k_gemm_tf32");
  return AOL_OK;
}

static int gemm_core_3x(const float* A, const float* B, float* C, const GemmShape& g, int64_t first, int64_t count,
                        cudaStream_t stream) {
  using namespace gemm;
  CUtensorMap ma, mb;
  int rc;
  if (g.a_kmajor) rc = make_map(&ma, A, g.K, g.M, g.lda, BK, x3::HALF_M, true);
  else rc = make_map(&ma, A, g.M, g.K, g.lda, 32, BK, false);
  if (rc) return rc;
  // form (read once per process): 2 = "regs" (256x256 pair tiles, two TMEM chunk accumulators,
  // running sum in registers; default), 1 = "wide" (256x256, one accumulator + TMEM running
  // sum), 0 = "narrow" (256x128, two 128-column accumulators + TMEM running sum) -- same bits
  static const int form = [] {
    const char* f = getenv("AOL_3XTF32_FORM");
    const char* w = getenv("AOL_3XTF32_WIDE");
    if (f) return !strcmp(f, "narrow") ? 0 : !strcmp(f, "wide") ? 1 : 2;
    return (w && w[0] == '0') ? 0 : 2;
  }();
  const bool wide = form != 0;
  if (g.b_kmajor) rc = make_map(&mb, B, g.K, g.N, g.ldb, BK, wide ? x3w::HALF_N : x3::HALF_N, true);
  else rc = make_map(&mb, B, g.N, g.K, g.ldb, 32, BK, false);
  if (rc) return rc;
  Params p{};
  p.c = C;
  p.ldc = g.ldc;
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.first = first;
  p.last = first + count - 1;
  p.m_lo = first / g.N;
  p.m_hi = p.last / g.N;
  p.row_base = g.a_kmajor ? p.m_lo : (p.m_lo & ~int64_t(31));
  p.m_tiles = (int)((p.m_hi - p.row_base + x3::BM) / x3::BM);
  p.n_tiles = (int)((g.N + (wide ? x3w::BN : x3::BN) - 1) / (wide ? x3w::BN : x3::BN));
  p.k_blocks = (int)((g.K + BK - 1) / BK);
  p.num_tiles = p.m_tiles * p.n_tiles;
  p.c_vec = ((uintptr_t)C % 16 == 0) && (g.ldc % 4 == 0);
  p.group_m = 8;
  const char* ck = getenv("AOL_3XTF32_CHUNK");          // K elements per TMEM chunk (multiple of 32)
  p.chunk_kb = ck ? (atoi(ck) / BK > 0 ? atoi(ck) / BK : 1) : (wide ? x3w::CHUNK_KB : x3::CHUNK_KB);
  const char* hr = getenv("AOL_3XTF32_HI");
  p.hi_round = hr ? (hr[0] != '0') : 0;
  void (*k)(const CUtensorMap, const CUtensorMap, Params);
  if (form == 2) {
    if (g.a_kmajor) k = g.b_kmajor ? x3r::k_gemm_3xtf32_regs<true, true> : x3r::k_gemm_3xtf32_regs<true, false>;
    else k = g.b_kmajor ? x3r::k_gemm_3xtf32_regs<false, true> : x3r::k_gemm_3xtf32_regs<false, false>;
  } else if (wide) {
    if (g.a_kmajor) k = g.b_kmajor ? x3w::k_gemm_3xtf32_wide<true, true> : x3w::k_gemm_3xtf32_wide<true, false>;
    else k = g.b_kmajor ? x3w::k_gemm_3xtf32_wide<false, true> : x3w::k_gemm_3xtf32_wide<false, false>;
  } else {
    if (g.a_kmajor) k = g.b_kmajor ? x3::k_gemm_3xtf32_pair<true, true> : x3::k_gemm_3xtf32_pair<true, false>;
    else k = g.b_kmajor ? x3::k_gemm_3xtf32_pair<false, true> : x3::k_gemm_3xtf32_pair<false, false>;
  }
  const int smem = (int)(form == 2 ? x3r::SMEM_BYTES : wide ? x3w::SMEM_BYTES : x3::SMEM_BYTES);
  AOL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int sms = kNumSMs;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pairs = p.num_tiles < sms / 2 ? p.num_tiles : sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(form == 2 ? x3r::NUM_THREADS : wide ? x3w::NUM_THREADS : x3::NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AOL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, ma, mb, p));
  AOL_LAUNCH_CHECK(form == 2 ? "k_gemm_3xtf32_regs" : wide ? "k_gemm_3xtf32_wide" : "k_gemm_3xtf32_pair");
  return AOL_OK;
}

}  // namespace aol
