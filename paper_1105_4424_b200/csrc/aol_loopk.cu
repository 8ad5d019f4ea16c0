// A whole LoopStep (refexec.py:525-541) as ONE persistent cooperative kernel.
//
// The loop body of identity ops (copy/sub/scale/axpy/spmv_csr/dot_partial and the host
// scalar ops div/neg/rel_residual) is passed as a small program.  One CTA per SM runs
// it until relres <= tol or max_iter, so there is no launch and no host round trip per
// iteration.  Three rules keep every value bit-identical to the per-op kernels:
//
//  * element mapping: every vector op (and every dot) walks [first, first+count) in the
//    dot's fixed 1024 x 256 "virtual block" order.  Virtual block vb is run by one
//    256-thread sub-block, and thread t of vb touches first + vb*256 + t + k*262144.
//    So a value written by one elementwise op is re-read by the same thread.
//  * grid barriers (cooperative groups) are placed by a host-side hazard pass (below).
//    A barrier goes only before an op that re-reads a vector with a different mapping
//    (spmv's x gather, or a different `first`), or overwrites one that was read that way.
//    A dot always needs one barrier between its partials and the final tree.
//  * scalars: every CTA keeps every scalar port in shared memory (as the port dtype,
//    widened) and runs the dot final tree and the scalar ops redundantly.  Results are
//    identical everywhere, so scalars never need a barrier; CTA 0 writes them back.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "aol_common.cuh"
#include "aol_ident.cuh"

namespace cg = cooperative_groups;

namespace aol {

constexpr int kLoopMaxOps = 128;
constexpr int kLoopMaxGroups = 96;
constexpr int kLoopMaxPorts = 32;
constexpr int kLoopMaxParts = 8;
constexpr int kLoopSub = 4;                   // 256-thread sub-blocks per CTA
constexpr int kLoopThreads = 256 * kLoopSub;

struct LOp {
  int op, n_scalars, part, n_parts, dot;
  int sell;                                   // spmv: index into LProg::sell, or -1 (CSR rows)
  int reuse, reuse_it;                        // dot: take dot `reuse`'s value from iteration reuse_it on
  int level;                                  // scalar op: dependency level inside its group
  int port[6];
};

// An spmv matrix the body never writes, re-laid out once per call as SELL-32: slice s holds
// rows first+32s .. first+32s+31 of the op's range, entry k of lane l at base[s] + 32k + l.
// A warp's 32 rows then load their k-th entries as one coalesced access instead of 32 lines
// 216 B apart (tools/micro/sell.cu: 16.4 -> 7.6 us per 27-point spmv); the row sum still runs
// k = 0, 1, ... left to right, so results are the CSR rows' bit for bit.
constexpr int kLoopMaxSell = 4;
struct LSell {
  const int64_t* base;
  const void* colidx;
  const void* values;
};

// A group: consecutive vector ops over one launch range that need no barrier between them
// (each thread re-reads only what it wrote), optionally closed by a dot.  Or a run of host
// scalar ops.
struct LGroup {
  int barrier, op0, n_ops, scalar, dot;
  int levels;                                 // scalar group: dependency levels (ops of one level run in parallel)
  int64_t first, count;
};

struct LProg {
  int n_groups, n_ports, relres;
  double tol;
  int64_t max_iter;
  unsigned scalar_mask;                       // bit p: port p is a scalar (lives in smem)
  double* part;                               // [2][64][kDotBlocks] partials
  int64_t* state;                             // iterations, relres (bits), converged
  unsigned* ticket;                           // [2][64] arrivals per dot
  unsigned long long* result;                 // [2][64] published dot values (kSlotEmpty: not yet)
  unsigned long long* arrive;                 // [64] monotonic arrivals per dot (dot_mode 1), [64] barriers
  int dot_mode;                               // 0: last CTA reduces and publishes; 1: every CTA reduces
  int barrier_mode;                           // 0: cooperative-groups grid.sync; 1: arrival counter
  unsigned long long* prof;                   // AOL_LOOP_PROFILE: ns per group, CTA 0's view
  unsigned backoff_ns;                        // sleep between polls of a dot's flag
  LSell sell[kLoopMaxSell];
  LGroup groups[kLoopMaxGroups];
  LOp ops[kLoopMaxOps];
  void* ports[kLoopMaxPorts];
};

constexpr unsigned long long kSlotEmpty = ~0ull;   // sentinel NaN: never an arithmetic result

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void sub_sync(int sub) {
  asm volatile("bar.sync %0, 256;" ::"r"(sub + 1) : "memory");
}

// one SELL-32 row: entries at b, b+32, b+64, ...; batches of 4 loads in flight, adds in order
template <typename T, typename I>
__device__ __forceinline__ T sell_row(const I* sc, const T* sv, const T* x, int64_t b, int len) {
  T acc = T(0);
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    I c[4];
    T v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = sc[b + 32 * (k + u)];
      v[u] = sv[b + 32 * (k + u)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  for (; k < len; ++k) acc = add_rn(acc, mul_rn(sv[b + 32 * k], x[sc[b + 32 * k]]));
  return acc;
}

// SELL build, step 1: 32 x (longest row) entries per slice (one warp per slice)
template <typename I>
__global__ void k_sell_width(const I* __restrict__ rowptr, int64_t first, int64_t count, int64_t* __restrict__ width) {
  const int64_t ns = (count + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < ns;
       s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = s * 32 + lane;
    int64_t len = r < count ? (int64_t)(rowptr[first + r + 1] - rowptr[first + r]) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) width[s] = 32 * len;
  }
}

// step 2: exclusive scan of the slice widths into base[0..ns] (one CTA, ns small)
__global__ void __launch_bounds__(1024) k_sell_scan(const int64_t* __restrict__ width, int64_t ns,
                                                    int64_t* __restrict__ base) {
  __shared__ int64_t part[1024];
  const int64_t per = (ns + 1023) / 1024, lo = threadIdx.x * per, hi = min(ns, lo + per);
  int64_t sum = 0;
  for (int64_t s = lo; s < hi; ++s) sum += width[s];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t s = lo; s < hi; ++s) {
    base[s] = run;
    run += width[s];
  }
  if (threadIdx.x == 1023) base[ns] = part[1023];
}

// step 3: scatter every row's entries into its slice, in row order
template <typename T, typename I>
__global__ void k_sell_fill(const I* __restrict__ rowptr, const I* __restrict__ colidx, const T* __restrict__ values,
                            int64_t first, int64_t count, const int64_t* __restrict__ base, I* __restrict__ sc,
                            T* __restrict__ sv) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q0 = rowptr[first + r], q1 = rowptr[first + r + 1];
    const int64_t b = base[r >> 5] + (r & 31);
    for (int64_t q = q0; q < q1; ++q) {
      sc[b + 32 * (q - q0)] = colidx[q];
      sv[b + 32 * (q - q0)] = values[q];
    }
  }
}

template <typename T, typename I>
__global__ void __launch_bounds__(kLoopThreads, 1) k_loop_persistent(const __grid_constant__ LProg P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sc[kLoopMaxPorts + kLoopMaxParts];
  __shared__ double red[kLoopSub][8];
  __shared__ double gred[32];
  __shared__ double dval[64];                 // each dot's final-tree value, for reuse
  __shared__ int s_last;
  const int sub = threadIdx.x >> 8, t = threadIdx.x & 255, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * kLoopSub + sub, nslots = gridDim.x * kLoopSub;
  const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
  // the program lives in shared memory: the interpreter's dependent lookups (op -> port ->
  // pointer) would otherwise be a chain of constant-cache misses per op
  __shared__ LGroup s_groups[kLoopMaxGroups];
  __shared__ LOp s_ops[kLoopMaxOps];
  __shared__ void* s_ports[kLoopMaxPorts];
  {
    const int* src = reinterpret_cast<const int*>(P.groups);
    int* dst = reinterpret_cast<int*>(s_groups);
    for (int i = threadIdx.x; i < (int)(sizeof(LGroup) / 4) * P.n_groups; i += blockDim.x) dst[i] = src[i];
    src = reinterpret_cast<const int*>(P.ops);
    dst = reinterpret_cast<int*>(s_ops);
    for (int i = threadIdx.x; i < (int)(sizeof(P.ops) / 4); i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x < kLoopMaxPorts) s_ports[threadIdx.x] = P.ports[threadIdx.x];
  }
  if (threadIdx.x < P.n_ports && ((P.scalar_mask >> threadIdx.x) & 1u))
    sc[threadIdx.x] = (double)((const T*)P.ports[threadIdx.x])[0];
  __syncthreads();

  int64_t it = 0;
  unsigned long long n_barriers = 0;
  int parity = 0;
  double relres = 0.0;
  int converged = 0;
  unsigned long long t_prev = 0;
  if (P.prof && writer) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prev));
  for (;;) {
    for (int gi = 0; gi < P.n_groups; ++gi) {
      const LGroup& G = s_groups[gi];
      if (P.prof && writer && gi > 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        P.prof[gi - 1] += now - t_prev;
        t_prev = now;
      }
      unsigned long long t_grp = 0;
      if (P.prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_grp));
      if (G.barrier) {
        if (P.barrier_mode == 1) {
          // the dots' arrival counter as a grid barrier: release-add, acquire-poll the total
          __syncthreads();
          ++n_barriers;
          if (threadIdx.x == 0) {
            unsigned long long* ctr = P.arrive + 64;
            const unsigned long long target = (unsigned long long)gridDim.x * n_barriers;
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
            uint32_t polls = 0;
            while (ld_acquire_u64(ctr) < target) {
              if (++polls == (1u << 31)) __trap();
              __nanosleep(P.backoff_ns);
            }
          }
          __syncthreads();
        } else {
          grid.sync();
        }
      }
      if (G.scalar) {                                   // host scalar ops, redundantly per CTA
        // lane k of warp 0 runs op op0+k; ops of one dependency level run side by side
        if (threadIdx.x < G.n_ops) {
          const LOp& o = s_ops[G.op0 + threadIdx.x];
          for (int lv = 0; lv < G.levels; ++lv) {
            if (o.level == lv) {
              double z;
              int out;
              if (o.op == AOL_OP_SCALAR_NEG) {
                z = (double)(-(T)sc[o.port[0]]);
                out = o.port[1];
              } else if (o.op == AOL_OP_SCALAR_DIV) {
                z = (double)(T)(sc[o.port[0]] / sc[o.port[1]]);
                out = o.port[2];
              } else {
                z = (double)(T)(sqrt(sc[o.port[0]]) / sqrt(sc[o.port[1]]));
                out = o.port[2];
              }
              sc[out] = z;
              if (blockIdx.x == 0) ((T*)s_ports[out])[0] = (T)z;
            }
            __syncwarp(G.n_ops >= 32 ? 0xffffffffu : (1u << G.n_ops) - 1u);
          }
        }
        __syncthreads();
        continue;
      }
      const int last = G.op0 + G.n_ops;
      // virtual blocks past the range hold no elements: their dot partials stay +0.0
      const int vb_end = (int)std::min<int64_t>(kDotBlocks, (G.count + 255) / 256);
      const int64_t end = G.first + G.count;
#define LOOP_EW(i)                                                                      \
  for (int vb = slot; vb < vb_end; vb += nslots)                                        \
    for (int64_t i = G.first + (int64_t)vb * 256 + t; i < end; i += (int64_t)kDotBlocks * 256)
      for (int k = G.op0; k < last; ++k) {
        const LOp& o = s_ops[k];
        switch (o.op) {
          case AOL_OP_COPY: {
            const T* src = (const T*)s_ports[o.port[0]];
            T* dst = (T*)s_ports[o.port[1]];
            LOOP_EW(i) dst[i] = src[i];
            break;
          }
          case AOL_OP_SUB: {
            const T* x = (const T*)s_ports[o.port[0]];
            const T* y = (const T*)s_ports[o.port[1]];
            T* z = (T*)s_ports[o.port[2]];
            LOOP_EW(i) z[i] = sub_rn(x[i], y[i]);
            break;
          }
          case AOL_OP_SCALE: {
            T* y = (T*)s_ports[o.port[0]];
            const T a = (T)sc[o.port[1]];
            LOOP_EW(i) y[i] = mul_rn(y[i], a);
            break;
          }
          case AOL_OP_AXPY: {
            T* y = (T*)s_ports[o.port[0]];
            const T* x = (const T*)s_ports[o.port[1]];
            if (o.n_scalars) {
              const T a = (T)sc[o.port[2]];
              LOOP_EW(i) y[i] = add_rn(y[i], mul_rn(a, x[i]));
            } else {
              LOOP_EW(i) y[i] = add_rn(y[i], x[i]);
            }
            break;
          }
          case AOL_OP_SPMV_CSR: {
            const I* rowptr = (const I*)s_ports[o.port[0]];
            const I* colidx = (const I*)s_ports[o.port[1]];
            const T* values = (const T*)s_ports[o.port[2]];
            const T* x = (const T*)s_ports[o.port[3]];
            T* y = (T*)s_ports[o.port[4]];
            if (o.sell >= 0) {
              const LSell& S = P.sell[o.sell];
              const I* sc = (const I*)S.colidx;
              const T* sv = (const T*)S.values;
              LOOP_EW(i) {
                const int64_t r = i - G.first;
                y[i] = sell_row(sc, sv, x, S.base[r >> 5] + (r & 31), (int)(rowptr[i + 1] - rowptr[i]));
              }
            } else {
              LOOP_EW(i) y[i] = csr_row(colidx, values, x, (int64_t)rowptr[i], (int64_t)rowptr[i + 1]);
            }
            break;
          }
          case AOL_OP_DOT_PARTIAL: {                  // k_dot's per-block partials, exactly
            if (o.reuse >= 0 && it >= o.reuse_it) break;
            const T* a = (const T*)s_ports[o.port[0]];
            const T* b = (const T*)s_ports[o.port[1]];
            double* part = P.part + ((size_t)parity * 64 + o.dot) * kDotBlocks;
            for (int vb = slot; vb < vb_end; vb += nslots) {
              double acc = 0.0;
              for (int64_t i = G.first + (int64_t)vb * 256 + t; i < end; i += (int64_t)kDotBlocks * 256)
                acc = fma((double)a[i], (double)b[i], acc);
              acc = warp_sum(acc);
              if (lane == 0) red[sub][t >> 5] = acc;
              sub_sync(sub);
              if (t < 32) {
                double w = t < 8 ? red[sub][t] : 0.0;
                w = warp_sum(w);
                if (t == 0) part[vb] = w;
              }
              sub_sync(sub);
            }
            break;
          }
          default: break;
        }
      }
#undef LOOP_EW
      if (!G.dot) continue;
      const LOp& o = s_ops[last - 1];
      const double* part = P.part + ((size_t)parity * 64 + o.dot) * kDotBlocks;
      const int cell = parity * 64 + o.dot;
      unsigned long long t1 = 0, t2 = 0;
      if (P.prof && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicAdd(P.prof + kLoopMaxGroups + 2 * blockIdx.x, t1 - t_grp);
      }
      const bool reused = o.reuse >= 0 && it >= o.reuse_it;
      if (reused) {
        if (threadIdx.x == 0) gred[0] = dval[o.reuse];
      } else if (P.dot_mode == 1) {
        // Arrival count instead of a grid barrier, and no publish hop: every CTA adds itself
        // to the dot's monotonic counter (release), waits until all gridDim.x arrivals of
        // this iteration are in (acquire), then runs k_dot's final tree itself over the 1024
        // partials.  Same inputs, same order: every CTA gets the same bits.
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long* ctr = P.arrive + o.dot;
          const unsigned long long target = (unsigned long long)gridDim.x * (unsigned long long)(it + 1);
          asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
          uint32_t polls = 0;
          while (ld_acquire_u64(ctr) < target) {
            if (++polls == (1u << 31)) __trap();                // a lost arrival: fail, never hang
            __nanosleep(P.backoff_ns);
          }
        }
        __syncthreads();
        {                                             // 32 warps: one 32-partial group each
          static_assert(kLoopThreads / 32 == kDotBlocks / 32, "one warp per partial group");
          double w = __ldcg(part + warp * 32 + lane);
          w = warp_sum(w);
          if (lane == 0) gred[warp] = w;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
          const double w = warp_sum(gred[lane]);
          if (lane == 0) gred[0] = w;
        }
      } else {
      // Ticket instead of a grid barrier: the last CTA to arrive runs k_dot's final tree
      // once and publishes the value into an 8-byte slot holding a sentinel NaN (all ones:
      // arithmetic only produces the canonical NaN); the others poll that slot with acquire
      // loads and get the value in the same load.  The slot of the other parity (read by
      // everyone one iteration ago, written again one iteration ahead) is re-armed first.
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(P.ticket + cell, 1u) == gridDim.x - 1;
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        if (warp < 8) {
          for (int g = warp; g < kDotBlocks / 32; g += 8) {
            double w = __ldcg(part + g * 32 + lane);
            w = warp_sum(w);
            if (lane == 0) gred[g] = w;
          }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
          const double w = warp_sum(gred[lane]);
          if (lane == 0) {
            P.ticket[cell] = 0;
            P.result[cell ^ 64] = kSlotEmpty;
            __threadfence();
            st_release_u64(P.result + cell, (unsigned long long)__double_as_longlong(w));
            gred[0] = w;
          }
        }
      } else if (threadIdx.x == 0) {
        unsigned long long v;
        uint32_t polls = 0;
        while ((v = ld_acquire_u64(P.result + cell)) == kSlotEmpty) {
          if (++polls == (1u << 31)) __trap();                  // a lost publish: fail, never hang
          __nanosleep(P.backoff_ns);
        }
        gred[0] = __longlong_as_double((long long)v);
      }
      }
      __syncthreads();
      if (threadIdx.x == 0) dval[o.dot] = gred[0];
      if (P.prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
      if (threadIdx.x < 32) {
        const double w = gred[0];
        if (lane == 0) {
          const double pv = (double)(T)__dadd_rn(0.0, w);
          if (o.n_parts == 1) {
            sc[o.port[2]] = pv;
            if (writer) ((T*)s_ports[o.port[2]])[0] = (T)pv;
          } else {
            sc[kLoopMaxPorts + o.part] = pv;
            if (o.part == o.n_parts - 1) {             // refexec.py:483-486: 0.0 + p0 + p1 ... in order
              double total = 0.0;
              for (int q = 0; q < o.n_parts; ++q) total = __dadd_rn(total, sc[kLoopMaxPorts + q]);
              sc[o.port[2]] = (double)(T)total;
              if (writer) ((T*)s_ports[o.port[2]])[0] = (T)total;
            }
          }
        }
      }
      __syncthreads();
      if (P.prof && threadIdx.x == 0) {
        unsigned long long t3;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
        atomicAdd(P.prof + kLoopMaxGroups + 2 * blockIdx.x + 1, t3 - t2);
      }
    }
    if (P.prof && writer) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      P.prof[P.n_groups - 1] += now - t_prev;
      t_prev = now;
    }
    ++it;
    parity ^= 1;
    relres = sc[P.relres];
    if (relres <= P.tol) {
      converged = 1;
      break;
    }
    if (it >= P.max_iter) break;
  }
  if (writer) {
    P.state[0] = it;
    P.state[1] = __double_as_longlong(relres);
    P.state[2] = converged;
  }
}

// -- host side: program checks, grouping and the barrier (hazard) pass ---------------

namespace {

enum Acc { R = 0, W = 1, G = 2 };      // elementwise read / elementwise write / gather read
struct Access {
  int port;
  Acc mode;
  int arg;                             // operand position in aol_loop_op.port
};

// vector accesses of one op in evaluation order (reads before the write)
std::vector<Access> vector_accesses(const aol_loop_op& o) {
  switch (o.op) {
    case AOL_OP_COPY: return {{o.port[0], R, 0}, {o.port[1], W, 1}};
    case AOL_OP_SUB: return {{o.port[0], R, 0}, {o.port[1], R, 1}, {o.port[2], W, 2}};
    case AOL_OP_SCALE: return {{o.port[0], R, 0}, {o.port[0], W, 0}};
    case AOL_OP_AXPY: return {{o.port[0], R, 0}, {o.port[1], R, 1}, {o.port[0], W, 0}};
    case AOL_OP_SPMV_CSR:
      return {{o.port[0], G, 0}, {o.port[1], G, 1}, {o.port[2], G, 2}, {o.port[3], G, 3}, {o.port[4], W, 4}};
    case AOL_OP_DOT_PARTIAL: return {{o.port[0], R, 0}, {o.port[1], R, 1}};
    default: return {};
  }
}

std::vector<int> scalar_ports(const aol_loop_op& o) {
  switch (o.op) {
    case AOL_OP_SCALE: return {o.port[1]};
    case AOL_OP_AXPY: return o.n_scalars ? std::vector<int>{o.port[2]} : std::vector<int>{};
    case AOL_OP_DOT_PARTIAL: return {o.port[2]};
    case AOL_OP_SCALAR_DIV: return {o.port[0], o.port[1], o.port[2]};
    case AOL_OP_SCALAR_NEG: return {o.port[0], o.port[1]};
    case AOL_OP_REL_RESIDUAL: return {o.port[0], o.port[1], o.port[2]};
    default: return {};
  }
}

bool is_scalar_op(int op) {
  return op == AOL_OP_SCALAR_DIV || op == AOL_OP_SCALAR_NEG || op == AOL_OP_REL_RESIDUAL;
}

struct Seen {
  int port;
  Acc mode;
  int64_t key;
};

// Does access `a` (under launch key `key`) race with an access made since the last barrier?
// Same-key elementwise accesses are the same thread's; everything else crosses threads.
bool conflicts(const std::vector<Seen>& seen, const Access& a, int64_t key) {
  for (const Seen& s : seen) {
    if (s.port != a.port) continue;
    if (a.mode == G && s.mode == W) return true;
    if (a.mode == R && s.mode == W && s.key != key) return true;
    if (a.mode == W && (s.mode == G || s.key != key)) return true;
  }
  return false;
}

struct Plan {
  std::vector<LGroup> groups;
  std::vector<LOp> ops;
};

// Split the body into groups and mark the groups that must start with a grid barrier.
// Barrier flags are decided over two passes of the body, because the loop wraps.
// Dot reuse (common-subexpression elimination that keeps the bits): dot j may take the
// final-tree value of the nearest earlier dot k (cyclically; from iteration 1 on when k
// comes later in the body) over the same ports and launch range when no op between them
// writes either vector.  Same inputs in the same fixed order give the same value, so the
// second reduction, its arrival wait and its final tree are skipped.  CG's dot_rr(r, r)
// reuses the previous iteration's dot_rrn(r, r) (cg.gmodel).
struct Reuse {
  int from = -1, from_it = 0;
};

static bool writes_port(const aol_loop_op& o, int port) {
  for (const Access& a : vector_accesses(o))
    if (a.mode == W && a.port == port) return true;
  return false;
}

std::vector<Reuse> plan_dot_reuse(const aol_loop_op* ops, int n) {
  std::vector<Reuse> r(n);
  const char* env = getenv("AOL_LOOP_DOT_REUSE");
  if (env && env[0] == '0') return r;
  for (int j = 0; j < n; ++j) {
    const aol_loop_op& oj = ops[j];
    if (oj.op != AOL_OP_DOT_PARTIAL) continue;
    for (int step = 1; step < n; ++step) {
      const int k = (j - step + n) % n;
      const aol_loop_op& ok = ops[k];
      if (ok.op == AOL_OP_DOT_PARTIAL && ok.port[0] == oj.port[0] && ok.port[1] == oj.port[1] &&
          ok.first == oj.first && ok.count == oj.count && ok.part == oj.part && ok.n_parts == oj.n_parts) {
        r[j].from = k;
        r[j].from_it = k > j ? 1 : 0;
        break;
      }
      if (writes_port(ok, oj.port[0]) || writes_port(ok, oj.port[1])) break;
    }
  }
  return r;
}

Plan plan_groups(const aol_loop_op* ops, int n, const std::vector<Reuse>& reuse) {
  Plan pl;
  // 1. grouping (independent of the wrap): a new group at every scalar op, key change,
  //    in-group race, and after every dot
  {
    std::vector<Seen> in_group;
    LGroup cur{};
    bool open = false;
    auto close = [&]() {
      if (open) pl.groups.push_back(cur);
      open = false;
      in_group.clear();
    };
    for (int k = 0; k < n; ++k) {
      const aol_loop_op& o = ops[k];
      LOp d{};
      d.op = o.op;
      d.n_scalars = o.n_scalars;
      d.part = o.part;
      d.n_parts = o.n_parts;
      for (int q = 0; q < 6; ++q) d.port[q] = o.port[q];
      if (is_scalar_op(o.op)) {
        close();
        if (!pl.groups.empty() && pl.groups.back().scalar && pl.groups.back().op0 + pl.groups.back().n_ops == k) {
          pl.groups.back().n_ops++;
          pl.ops.push_back(d);
          continue;
        }
        LGroup g{};
        g.scalar = 1;
        g.op0 = k;
        g.n_ops = 1;
        pl.groups.push_back(g);
        pl.ops.push_back(d);
        continue;
      }
      const std::vector<Access> acc = vector_accesses(o);
      bool fresh = !open || cur.first != o.first || cur.count != o.count;
      if (!fresh)
        for (const Access& a : acc) fresh = fresh || conflicts(in_group, a, o.first);
      if (fresh) {
        close();
        cur = LGroup{};
        cur.op0 = k;
        cur.first = o.first;
        cur.count = o.count;
        open = true;
      }
      for (const Access& a : acc) in_group.push_back({a.port, a.mode, o.first});
      cur.n_ops = k - cur.op0 + 1;
      pl.ops.push_back(d);
      if (o.op == AOL_OP_DOT_PARTIAL) {
        cur.dot = 1;
        close();
      }
    }
    close();
  }
  // 2. barriers, over body + body
  std::vector<Seen> seen;
  for (int pass = 0; pass < 2; ++pass) {
    for (LGroup& g : pl.groups) {
      if (g.scalar) continue;
      std::vector<Access> acc;
      for (int k = g.op0; k < g.op0 + g.n_ops; ++k)
        for (const Access& a : vector_accesses(ops[k])) acc.push_back(a);
      bool need = false;
      for (const Access& a : acc) need = need || conflicts(seen, a, g.first);
      if (need) {
        g.barrier = 1;
        seen.clear();
      }
      for (const Access& a : acc) seen.push_back({a.port, a.mode, g.first});
      // the dot's own barrier (a reused dot synchronises nothing)
      if (g.dot && reuse[g.op0 + g.n_ops - 1].from < 0) seen.clear();
    }
  }
  return pl;
}

// SELL-32 copy of one spmv matrix (k_sell_width -> k_sell_scan -> k_sell_fill) into the
// device's slot buffers; one synchronous read of the total size.
struct SellBufs {
  void* meta = nullptr;
  size_t meta_cap = 0;
  void* data = nullptr;
  size_t data_cap = 0;
};

static int grow(void*& p, size_t& cap, size_t need) {
  if (need <= cap) return AOL_OK;
  if (p) AOL_CUDA_CHECK(cudaFree(p));
  p = nullptr;
  cap = 0;
  AOL_CUDA_CHECK(cudaMalloc(&p, need));
  cap = need;
  return AOL_OK;
}

template <typename T, typename I>
static int build_sell(const aol_loop_op& o, void* const* ports, SellBufs& b, LSell& out, cudaStream_t s) {
  const I* rowptr = static_cast<const I*>(ports[o.port[0]]);
  const int64_t ns = (o.count + 31) / 32;
  int rc = grow(b.meta, b.meta_cap, (size_t)(2 * ns + 1) * sizeof(int64_t));
  if (rc) return rc;
  int64_t* width = static_cast<int64_t*>(b.meta);
  int64_t* base = width + ns;
  k_sell_width<I><<<(unsigned)std::min<int64_t>((ns + 7) / 8, 4096), 256, 0, s>>>(rowptr, o.first, o.count, width);
  AOL_LAUNCH_CHECK("k_sell_width");
  k_sell_scan<<<1, 1024, 0, s>>>(width, ns, base);
  AOL_LAUNCH_CHECK("k_sell_scan");
  int64_t total = 0;
  AOL_CUDA_CHECK(cudaMemcpyAsync(&total, base + ns, sizeof(total), cudaMemcpyDeviceToHost, s));
  AOL_CUDA_CHECK(cudaStreamSynchronize(s));
  const size_t sc_bytes = ((size_t)total * sizeof(I) + 255) / 256 * 256;
  rc = grow(b.data, b.data_cap, sc_bytes + (size_t)total * sizeof(T) + 256);
  if (rc) return rc;
  I* sc = static_cast<I*>(b.data);
  T* sv = reinterpret_cast<T*>(static_cast<char*>(b.data) + sc_bytes);
  k_sell_fill<T, I><<<(unsigned)std::min<int64_t>((o.count + 255) / 256, 4096), 256, 0, s>>>(
      rowptr, static_cast<const I*>(ports[o.port[1]]), static_cast<const T*>(ports[o.port[2]]), o.first, o.count,
      base, sc, sv);
  AOL_LAUNCH_CHECK("k_sell_fill");
  out.base = base;
  out.colidx = sc;
  out.values = sv;
  return AOL_OK;
}

}  // namespace

}  // namespace aol

using namespace aol;

namespace aol {
// persistent-loop scratch, one block per device, allocated on first use (see below)
static std::mutex g_loop_locks[64];
static char* g_loop_scratch[64] = {nullptr};
static int g_loop_fits[64] = {0};

int release_loop_scratch() {
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < 64; ++d) {
    std::lock_guard<std::mutex> lock(g_loop_locks[d]);
    if (!g_loop_scratch[d]) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    cudaFree(g_loop_scratch[d]);
    g_loop_scratch[d] = nullptr;
  }
  cudaSetDevice(cur);
  return 0;
}
}  // namespace aol

extern "C" int aol_loop_persistent(const aol_loop_op* ops, int n_ops, void* const* ports, int n_ports, int dtype,
                                   int index_dtype, int relres_port, double tol, int64_t max_iter, void* stream,
                                   int64_t* iterations, double* final_relres, int* converged) {
  const auto host_t0 = std::chrono::steady_clock::now();
  if (!ops || !ports || n_ops < 1 || max_iter < 1) return fail(AOL_EINVAL, "aol_loop_persistent: bad arguments");
  if (n_ops > kLoopMaxOps || n_ports > kLoopMaxPorts)
    return fail(AOL_EUNSUPPORTED, "loop body too large for the persistent interpreter");
  if (dtype != AOL_F32 && dtype != AOL_F64) return fail(AOL_EUNSUPPORTED, "persistent loop needs float32/float64");
  if (index_dtype != AOL_I32 && index_dtype != AOL_I64) return fail(AOL_EINVAL, "bad index dtype");
  if (relres_port < 0 || relres_port >= n_ports) return fail(AOL_EINVAL, "bad relres port");
  LProg P{};
  P.n_ports = n_ports;
  P.relres = relres_port;
  P.tol = tol;
  P.max_iter = max_iter;
  unsigned scalar = 0, vector = 0;
  int n_dots = 0;
  for (int k = 0; k < n_ops; ++k) {
    const aol_loop_op& o = ops[k];
    switch (o.op) {
      case AOL_OP_COPY: case AOL_OP_SUB: case AOL_OP_SCALE: case AOL_OP_AXPY: case AOL_OP_SPMV_CSR:
      case AOL_OP_DOT_PARTIAL: case AOL_OP_SCALAR_DIV: case AOL_OP_SCALAR_NEG: case AOL_OP_REL_RESIDUAL:
        break;
      default:
        return fail(AOL_EUNSUPPORTED, "op " + std::to_string(o.op) + " not in the persistent interpreter");
    }
    for (int q = 0; q < 6; ++q)
      if (o.port[q] >= n_ports) return fail(AOL_EINVAL, "port index out of range");
    if (o.first < 0 || o.count < 0) return fail(AOL_EINVAL, "bad launch range");
    if (o.op == AOL_OP_DOT_PARTIAL) {
      if (o.n_parts < 1 || o.n_parts > kLoopMaxParts || o.part < 0 || o.part >= o.n_parts)
        return fail(AOL_EUNSUPPORTED, "dot partial index out of range");
      if (n_dots >= 64) return fail(AOL_EUNSUPPORTED, "too many dots");
      ++n_dots;
    }
    for (const Access& a : vector_accesses(o)) {
      if (a.port < 0) return fail(AOL_EINVAL, "port index out of range");
      vector |= 1u << a.port;
    }
    for (int p : scalar_ports(o)) {
      if (p < 0) return fail(AOL_EINVAL, "port index out of range");
      scalar |= 1u << p;
    }
  }
  if (scalar & vector) return fail(AOL_EUNSUPPORTED, "a port is used both as a scalar and as a vector");
  if (!((scalar >> relres_port) & 1u)) return fail(AOL_EUNSUPPORTED, "relres is not a scalar of the body");
  for (int p = 0; p < n_ports; ++p)
    if (!ports[p]) return fail(AOL_EINVAL, "null port");
  const std::vector<Reuse> reuse = plan_dot_reuse(ops, n_ops);
  Plan pl = plan_groups(ops, n_ops, reuse);
  if ( (int)pl.groups.size() > kLoopMaxGroups)
    return fail(AOL_EUNSUPPORTED, "loop body does not fit the persistent interpreter");
  int dot = 0;
  unsigned written = 0;
  for (int k = 0; k < n_ops; ++k)
    for (const Access& a : vector_accesses(ops[k]))
      if (a.mode == W) written |= 1u << a.port;
  std::vector<int> dot_id(n_ops, 0);
  for (int k = 0; k < n_ops; ++k) {
    P.ops[k] = pl.ops[k];
    P.ops[k].dot = dot_id[k] = ops[k].op == AOL_OP_DOT_PARTIAL ? dot++ : 0;
    P.ops[k].sell = -1;
  }
  for (int k = 0; k < n_ops; ++k) {
    P.ops[k].reuse = reuse[k].from >= 0 ? dot_id[reuse[k].from] : -1;
    P.ops[k].reuse_it = reuse[k].from_it;
    P.ops[k].level = 0;
  }
  // scalar groups: an op's level is 1 + the deepest earlier op of its group it reads from
  for (size_t g = 0; g < pl.groups.size(); ++g) {
    LGroup& G = pl.groups[g];
    G.levels = 1;
    if (!G.scalar) continue;
    if (G.n_ops > 32) return fail(AOL_EUNSUPPORTED, "scalar run longer than a warp");
    for (int k = G.op0; k < G.op0 + G.n_ops; ++k) {
      const aol_loop_op& o = ops[k];
      const int n_in = o.op == AOL_OP_SCALAR_NEG ? 1 : 2;
      int lv = 0;
      for (int j = G.op0; j < k; ++j) {
        const aol_loop_op& p = ops[j];
        const int out = p.op == AOL_OP_SCALAR_NEG ? p.port[1] : p.port[2];
        for (int q = 0; q < n_in; ++q)
          if (o.port[q] == out) lv = std::max(lv, P.ops[j].level + 1);
        // an op overwriting what an earlier op of the group reads or writes goes after it
        const int my_out = o.op == AOL_OP_SCALAR_NEG ? o.port[1] : o.port[2];
        const int p_in = p.op == AOL_OP_SCALAR_NEG ? 1 : 2;
        for (int q = 0; q < p_in; ++q)
          if (p.port[q] == my_out) lv = std::max(lv, P.ops[j].level + 1);
        if (out == my_out) lv = std::max(lv, P.ops[j].level + 1);
      }
      P.ops[k].level = lv;
      G.levels = std::max(G.levels, lv + 1);
    }
  }
  for (size_t g = 0; g < pl.groups.size(); ++g) P.groups[g] = pl.groups[g];
  P.n_groups = (int)pl.groups.size();
  for (int p = 0; p < n_ports; ++p) P.ports[p] = ports[p];
  P.scalar_mask = scalar;
  {
    const char* b = getenv("AOL_LOOP_BACKOFF_NS");
    P.backoff_ns = b ? (unsigned)atoi(b) : 32u;
  }

  int dev = 0, coop = 0, per_sm = 0, sms = 0;
  AOL_CUDA_CHECK(cudaGetDevice(&dev));
  AOL_CUDA_CHECK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  AOL_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (!coop) return fail(AOL_EUNSUPPORTED, "device has no cooperative launch");
  void (*kern)(LProg);
  if (dtype == AOL_F64) kern = index_dtype == AOL_I64 ? k_loop_persistent<double, int64_t> : k_loop_persistent<double, int32_t>;
  else kern = index_dtype == AOL_I64 ? k_loop_persistent<float, int64_t> : k_loop_persistent<float, int32_t>;
  if (dev < 0 || dev >= 64) return fail(AOL_EUNSUPPORTED, "device index out of range");
  // per device: occupancy checked once, scratch allocated once (the call is synchronous and
  // holds the device's lock, so loops on one device never share scratch concurrently)
  std::lock_guard<std::mutex> lock(g_loop_locks[dev]);
  char** scratch_of = g_loop_scratch;
  int* fits_of = g_loop_fits;
  const int kid = (dtype == AOL_F64 ? 2 : 0) + (index_dtype == AOL_I64 ? 1 : 0);
  if (!((fits_of[dev] >> kid) & 1)) {
    AOL_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLoopThreads, 0));
    if (per_sm < 1) return fail(AOL_EUNSUPPORTED, "persistent loop kernel does not fit on an SM");
    fits_of[dev] |= 1 << kid;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t part_bytes = (size_t)2 * 64 * kDotBlocks * sizeof(double);
  const size_t prof_bytes = (kLoopMaxGroups + 2 * 1024) * sizeof(unsigned long long);
  const char* prof_env = getenv("AOL_LOOP_PROFILE");
  const bool profile = prof_env && prof_env[0] == '1';
  const size_t sync_bytes = 128 * (4 + 4 + 8) + 72 * 8;
  if (!scratch_of[dev]) AOL_CUDA_CHECK(cudaMalloc(&scratch_of[dev], part_bytes + 64 + sync_bytes + prof_bytes));
  char* scratch = scratch_of[dev];
  P.part = reinterpret_cast<double*>(scratch);
  P.state = reinterpret_cast<int64_t*>(scratch + part_bytes);
  P.ticket = reinterpret_cast<unsigned*>(scratch + part_bytes + 64);
  P.result = reinterpret_cast<unsigned long long*>(P.ticket + 256);
  AOL_CUDA_CHECK(cudaMemsetAsync(P.ticket, 0, 256 * sizeof(unsigned), s));
  AOL_CUDA_CHECK(cudaMemsetAsync(P.result, 0xff, 128 * sizeof(unsigned long long), s));
  P.arrive = P.result + 128;
  AOL_CUDA_CHECK(cudaMemsetAsync(P.arrive, 0, 65 * sizeof(unsigned long long), s));
  {
    const char* dm = getenv("AOL_LOOP_DOT");
    P.dot_mode = (dm && dm[0] == '0') ? 0 : 1;
    const char* bm = getenv("AOL_LOOP_BARRIER");
    P.barrier_mode = (bm && bm[0] == '0') ? 0 : 1;
  }
  AOL_CUDA_CHECK(cudaMemsetAsync(P.part, 0, part_bytes, s));
  P.prof = profile ? reinterpret_cast<unsigned long long*>(scratch + part_bytes + 64 + sync_bytes) : nullptr;
  // SELL-32 copies of the spmv matrices the body never writes (AOL_LOOP_SELL=0: CSR rows)
  {
    static SellBufs sell_bufs[64][kLoopMaxSell];
    const char* se = getenv("AOL_LOOP_SELL");
    int n_sell = 0;
    for (int k = 0; k < n_ops && !(se && se[0] == '0'); ++k) {
      const aol_loop_op& o = ops[k];
      if (o.op != AOL_OP_SPMV_CSR || o.count <= 0 || n_sell >= kLoopMaxSell) continue;
      if ((written >> o.port[0] & 1u) || (written >> o.port[1] & 1u) || (written >> o.port[2] & 1u)) continue;
      int rc;
      if (dtype == AOL_F64)
        rc = index_dtype == AOL_I64 ? build_sell<double, int64_t>(o, ports, sell_bufs[dev][n_sell], P.sell[n_sell], s)
                                    : build_sell<double, int32_t>(o, ports, sell_bufs[dev][n_sell], P.sell[n_sell], s);
      else
        rc = index_dtype == AOL_I64 ? build_sell<float, int64_t>(o, ports, sell_bufs[dev][n_sell], P.sell[n_sell], s)
                                    : build_sell<float, int32_t>(o, ports, sell_bufs[dev][n_sell], P.sell[n_sell], s);
      if (rc) return rc;
      P.ops[k].sell = n_sell++;
    }
  }
  if (profile) AOL_CUDA_CHECK(cudaMemsetAsync(P.prof, 0, prof_bytes, s));
  void* args[] = {&P};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const char* time_env = getenv("AOL_LOOP_TIME");
  const bool timed = profile || (time_env && time_env[0] == '1');
  if (timed) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, s);
  }
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(sms), dim3(kLoopThreads), args, 0, s);
  if (timed) cudaEventRecord(ev1, s);
  int64_t h[3] = {0, 0, 0};
  static unsigned long long prof[kLoopMaxGroups + 2 * 1024];
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, P.state, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && profile) e = cudaMemcpyAsync(prof, P.prof, prof_bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "aol_loop_persistent");
  count_launch();
  if (timed) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    fprintf(stderr, "aol_loop_persistent kernel %.3f ms, %lld iterations, %.2f us/iter; whole call %.3f ms\n", ms,
            (long long)h[0], 1e3 * ms / (h[0] ? h[0] : 1), host_ms);
  }
  if (profile) {
    for (int g = 0; g < P.n_groups; ++g) {
      const LGroup& G = P.groups[g];
      if (g == 0) {
        double mn = 1e30, mx = 0, sum = 0, tmn = 1e30, tmx = 0;
        int amx = 0;
        for (int c = 0; c < sms; ++c) {
          const double pre = prof[kLoopMaxGroups + 2 * c] * 1e-3 / h[0], tree = prof[kLoopMaxGroups + 2 * c + 1] * 1e-3 / h[0];
          mn = std::min(mn, pre);
          if (pre > mx) { mx = pre; amx = c; }
          sum += pre;
          tmn = std::min(tmn, tree);
          tmx = std::max(tmx, tree);
        }
        fprintf(stderr, "aol_loop_persistent dots, per CTA us/iter: before barrier min %.2f mean %.2f max %.2f (cta %d);"
                " tree min %.2f max %.2f\n", mn, sum / sms, mx, amx, tmn, tmx);
      }
      fprintf(stderr, "aol_loop_persistent group %2d: %s op0=%d n_ops=%d barrier=%d dot=%d  %.2f us/iter\n", g,
              G.scalar ? "scalar" : "vector", G.op0, G.n_ops, G.barrier, G.dot, h[0] ? prof[g] * 1e-3 / h[0] : 0.0);
    }
  }
  if (iterations) *iterations = h[0];
  if (final_relres) {
    double r;
    memcpy(&r, &h[1], sizeof(r));
    *final_relres = r;
  }
  if (converged) *converged = (int)h[2];
  return AOL_OK;
}
