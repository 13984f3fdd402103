// ozaki.cuh -- the FP64 contraction of the relaxation emulated on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Ozaki-style splitting with exact integer products:
//   every row r of A (and column c of B) is scaled by a power of two 2^e_r so
//   that |x| < 2^e_r, then cut into kOzS signed 8-bit digits
//       x = 2^e_r * sum_t d_t 2^(-6-7t) + rho,  |d_t| <= 64,  |rho| <= 2^(e_r-56)
//   (d_0 = rint(64 x'), each later digit the rint of the remainder times 128;
//   every remainder is exact in FP64).  Then
//       sum_k A[r,k] B[c,k] ~= 2^(e_r+e_c) sum_D 2^(-12-7D) C_D,
//       C_D = sum_{t+u=D} sum_k d^A_t[r,k] d^B_u[c,k]   (int32, exact),
//   keeping the diagonals D = t+u <= kOzS-1.  |C_D| <= kOzS * K * 64^2 < 2^31
//   for K <= 65 000, so the integer part is exact; the only rounding is the
//   FP64 recombination (small diagonals first) and the dropped tail
//   (~2^-55 of max|A_r| max|B_c| per product term).
//
// Kernel layout (one 128 x 64 output tile per CTA, K split over blockIdx.z):
//   warp 0 / lane 0: producer -- per 64-byte K block one 1-D bulk copy
//       (cp.async.bulk, the TMA engine's linear mode) of the A block and one
//       of the B block.  The digits are stored pre-tiled in global memory
//       as [tile][K block][digit][rows][64 B], each 64-byte row already
//       SWIZZLE_64B-permuted (16-byte chunk c of row r at c ^ ((r >> 1) & 3)),
//       i.e. exactly the UMMA K-major canonical shared-memory image: one
//       contiguous 64 KB (A) + 2-4 KB x 8 (B) copy per stage instead of one
//       TMA request per 64-byte row; two stages on full/empty mbarriers;
//   warp 1 / lane 0: MMA issuer -- for each A digit t and 32-column group,
//       one tcgen05.mma per K = 32 step whose B operand stacks the digits
//       u = 0 .. kOzS-1-t of the group (N = (kOzS-t)*32 <= 256): product
//       A_t B_u lands in TMEM column block t+u, the accumulator of its
//       diagonal (kOzS x 32 int32 columns per group: 512 TMEM columns for
//       64-column tiles).  8 MMAs of N <= 256 per K-step and group instead of
//       36 of N = 32; then tcgen05.commit to the stage's empty barrier;
//   all 4 warps: epilogue -- tcgen05.ld of the kOzS accumulators of their 32
//       TMEM lanes (rows), FP64 recombination, scale, store into the split's
//       slab (the consumers sum the slabs in order, as for the DMMA kernels).
#pragma once
#include <cstdint>

#include "gemm.cuh"  // EPI_STORE / EPI_DERIV, d_loss_deriv

namespace bnbg {

constexpr int kOzS = 8;           // digits per operand: 6 + 7*7 = 55 bits
constexpr int kOzBM = 128;        // UMMA M (rows of A per CTA)
constexpr int kOzBK = 64;         // K bytes per stage (SWIZZLE_64B row)
constexpr int kOzStages = 2;
constexpr int kOzThreads = 128;
constexpr int kOzASlab = kOzBM * kOzBK;  // 8 KB per digit
constexpr int kOzAStage = kOzS * kOzASlab;

// B rows are grouped by 32 columns: a group's digit slabs are contiguous,
// [digit][32 columns][64 B], so B_0 .. B_{S-1} of a group form one operand of
// up to 256 rows
constexpr int kOzG = 32;
constexpr int kOzGSlab = kOzG * kOzBK;  // 2 KB: one digit of one column group

// per column-tile width BN: 64, or 32 when the 64-wide tiles leave SMs idle
// (narrow batches, NN at c3)
template <int BN>
struct OzShape {
  static constexpr int BSlab = BN * kOzBK;  // 4 / 2 KB per digit
  static constexpr int StageBytes = kOzAStage + kOzS * BSlab;
  static constexpr int SmemBytes = kOzStages * StageBytes + 1024;  // + alignment slack
  static constexpr int TmemCols = kOzS * BN <= 256 ? 256 : 512;    // power of two
  static_assert(kOzS * BN <= TmemCols, "accumulators fit TMEM");
  static_assert(kOzASlab % 1024 == 0 && BSlab % 1024 == 0 && StageBytes % 1024 == 0,
                "swizzle atoms 1024-byte aligned");
};
constexpr int kOzSmemMax = OzShape<64>::SmemBytes;

struct OzArgs {
  const signed char* A;  // A digits, pre-tiled: [M tile][K block][digit][128][64 B]
  const signed char* B;  // B digits, pre-tiled: [N tile][K block][digit][BN][64 B]
  int nkb_total;         // K blocks per tile row of the layout
  const int* ea;     // per A row exponent
  const int* eb;     // per compact B column exponent
  int M, K;          // output rows, reduction length
  int ksplit;        // K per split (multiple of kOzBK)
  const int* d_ncols;  // active columns (device)
  const int* act;      // compact -> physical output column (nullptr: identity)
  double* C;
  int ldc;
  long long split_stride;
  // EPI_DERIV epilogue (NN: R = l'(X V), losses.hpp:65-69): y and the loss
  const double* y;
  int loss;
};

__device__ __forceinline__ unsigned oz_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void oz_bar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(oz_smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void oz_bar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "OZ_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra OZ_WAIT_%=;\n"
      "}\n" ::"r"(oz_smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void oz_bulk(void* dst, const void* src, unsigned bytes,
                                        unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          oz_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(oz_smem_u32(bar))
      : "memory");
}

// byte offset of (row r, byte kk) inside a pre-tiled digit slab of 64-byte
// rows: the SWIZZLE_64B permutation of the 16-byte chunks
__host__ __device__ __forceinline__ int oz_swz(int r, int kk) {
  return r * kOzBK + ((((kk >> 4) ^ (r >> 1)) & 3) << 4) + (kk & 15);
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B (rows of 64 bytes,
// 8-row atoms 512 bytes apart), sm_100 version 1.
__device__ __forceinline__ unsigned long long oz_desc(const void* p) {
  const unsigned long long addr = oz_smem_u32(p);
  unsigned long long d = 0;
  d |= (addr & 0x3FFFFull) >> 4;          // start address
  d |= 1ull << 16;                         // leading byte offset (unused, swizzled K-major)
  d |= (512ull >> 4) << 32;                // stride byte offset: 8 rows x 64 B
  d |= 1ull << 46;                         // version (sm_100)
  d |= 4ull << 61;                         // layout: SWIZZLE_64B
  return d;
}

// instruction descriptor: kind::i8, D s32, A/B signed, both K-major, M = 128, N
__host__ __device__ __forceinline__ constexpr unsigned oz_idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(n >> 3) << 17) |
         ((unsigned)(kOzBM >> 4) << 24);
}

__device__ __forceinline__ void oz_mma(unsigned tmem_d, unsigned long long da,
                                       unsigned long long db, unsigned idesc,
                                       unsigned accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void oz_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   oz_smem_u32(bar))
               : "memory");
}

template <int EPI, int BN>
__global__ void __launch_bounds__(kOzThreads, 1) k_ozaki_gemm(const __grid_constant__ OzArgs a) {
  using Sh = OzShape<BN>;
  extern __shared__ __align__(1024) unsigned char oz_raw[];
  __shared__ __align__(8) unsigned long long full_bar[kOzStages], empty_bar[kOzStages], done_bar;
  __shared__ unsigned tmem_base_s;
  // blockIdx.x walks the column tiles of one row tile: the CTAs that share
  // an A (X digits) tile run together and all but the first read it from L2
  const int ncols = *a.d_ncols;
  const int n0 = blockIdx.x * BN;
  if (n0 >= ncols) return;
  const int m0 = blockIdx.y * kOzBM;
  const int split = blockIdx.z;
  const int kbeg = split * a.ksplit;
  const int kend = min(a.K, kbeg + a.ksplit);
  const int nkb = (kend - kbeg + kOzBK - 1) / kOzBK;
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {  // TMEM: kOzS accumulators of BN int32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     oz_smem_u32(&tmem_base_s)),
                 "n"(Sh::TmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < kOzStages; ++s) {
      oz_bar_init(&full_bar[s], 1);
      oz_bar_init(&empty_bar[s], 1);
    }
    oz_bar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base_s;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kOzStages, u = kb / kOzStages;
      if (u > 0) oz_bar_wait(&empty_bar[s], (u - 1) & 1);  // MMAs of the last use done
      unsigned char* st = sm + s * Sh::StageBytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       oz_smem_u32(&full_bar[s])),
                   "r"((unsigned)Sh::StageBytes)
                   : "memory");
      const long long kbg = kbeg / kOzBK + kb;  // global K block
      oz_bulk(st, a.A + ((long long)blockIdx.y * a.nkb_total + kbg) * kOzAStage, kOzAStage,
              &full_bar[s]);
      oz_bulk(st + kOzAStage,
              a.B + ((long long)blockIdx.x * a.nkb_total + kbg) * (kOzS * Sh::BSlab),
              kOzS * Sh::BSlab, &full_bar[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kOzStages, u = kb / kOzStages;
      oz_bar_wait(&full_bar[s], u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* sa = sm + s * Sh::StageBytes;
      const unsigned char* sb = sa + kOzAStage;
      // digit-stacked N: for A digit t and a group of 32 columns, ONE MMA
      // against the B rows (digit u, column c) for u = 0 .. kOzS-1-t (N =
      // (kOzS-t)*32) lands every product A_t B_u in TMEM column block t+u =
      // the diagonal D it belongs to (accumulator [group][D][32 columns])
#pragma unroll 1
      for (int g = 0; g < BN / kOzG; ++g) {
#pragma unroll 1
        for (int t = 0; t < kOzS; ++t) {
          const unsigned idesc = oz_idesc((kOzS - t) * kOzG);
#pragma unroll
          for (int ks = 0; ks < kOzBK / 32; ++ks) {
            const unsigned long long da = oz_desc(sa + t * kOzASlab + ks * 32);
            const unsigned long long db = oz_desc(sb + g * kOzS * kOzGSlab + ks * 32);
            oz_mma(tmem + g * kOzS * kOzG + t * kOzG, da, db, idesc,
                   (kb > 0 || t > 0 || ks > 0) ? 1u : 0u);
          }
        }
      }
      oz_commit(&empty_bar[s]);  // frees the stage once these MMAs complete
    }
    oz_commit(&done_bar);
  }

  // ---- epilogue: all warps; warp w owns TMEM lanes (rows) 32w .. 32w+31 ----
  __syncwarp();  // lanes 1..31 of the producer / issuer warps park here, not spinning
  oz_bar_wait(&done_bar, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < a.M;
  const int er = row_ok ? a.ea[row] : 0;
  const double yv = (EPI == EPI_DERIV && row_ok) ? a.y[row] : 0.0;
  double* Cs = a.C + (size_t)split * a.split_stride;
#pragma unroll 1
  for (int cc = 0; cc < BN / 16; ++cc) {
    // the kOzS diagonals of this 16-column chunk in flight together, one wait
    unsigned v[kOzS][16];
#pragma unroll
    for (int D = 0; D < kOzS; ++D) {
      // column block of (group cc*16 / 32, diagonal D), 16-column half of it
      const unsigned taddr = tmem + ((unsigned)(warp * 32) << 16) +
                             (cc * 16 / kOzG) * kOzS * kOzG + D * kOzG + (cc * 16) % kOzG;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
          "%11, %12, %13, %14, %15}, [%16];"
          : "=r"(v[D][0]), "=r"(v[D][1]), "=r"(v[D][2]), "=r"(v[D][3]), "=r"(v[D][4]),
            "=r"(v[D][5]), "=r"(v[D][6]), "=r"(v[D][7]), "=r"(v[D][8]), "=r"(v[D][9]),
            "=r"(v[D][10]), "=r"(v[D][11]), "=r"(v[D][12]), "=r"(v[D][13]), "=r"(v[D][14]),
            "=r"(v[D][15])
          : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
#pragma unroll
    for (int D = kOzS - 1; D >= 0; --D) {  // smallest weights first
      const double w = ldexp(1.0, -12 - 7 * D);
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] += (double)(int)v[D][i] * w;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c = n0 + cc * 16 + i;
      if (row_ok && c < ncols) {
        const int col = a.act ? a.act[c] : c;
        const double sv = ldexp(acc[i], er + a.eb[c]);
        Cs[(size_t)col * a.ldc + row] = EPI == EPI_DERIV ? d_loss_deriv(a.loss, sv, yv) : sv;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(Sh::TmemCols));
}

// Digits of rows of a matrix, written pre-tiled and pre-swizzled (the
// producer's bulk-copy image): row r (physical rows[r] when rows != nullptr)
// has elements src[phys*ld_r + k*ld_k], k < K; rows are grouped in tiles of
// tile_rows, K in blocks of kOzBK bytes, and inside a tile in groups of
// group_rows: out[tile][kb][group][digit][group_rows][64 B] (A: one group of
// 128 rows; B: groups of kOzG columns).
// Rows r in [nrows, rows_pad) and k in [K, nkb*64) are zero.  exps[r].
// One CTA per row (rows_pad CTAs).
__global__ void k_oz_split_rows(const double* __restrict__ src, long long ld_r, long long ld_k,
                                const int* rows, int nrows, const int* d_nrows, int K, int nkb,
                                int tile_rows, int group_rows, signed char* __restrict__ out,
                                int* __restrict__ exps) {
  const int r = blockIdx.x;
  const int nr = d_nrows ? *d_nrows : nrows;
  const bool live = r < nr;
  const long long phys = live ? (rows ? rows[r] : r) : 0;
  const double* x = src + phys * ld_r;
  __shared__ double red[32];
  double mx = 0.0;
  if (live)
    for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmax(mx, fabs(x[(long long)k * ld_k]));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  int e = 0;
  if (mx > 0.0) {
    frexp(mx, &e);  // mx = f * 2^e, f in [0.5, 1): |x| < 2^e
  }
  if (live && threadIdx.x == 0) exps[r] = e;
  const int tile = r / tile_rows, rr = r % tile_rows;
  const int grp = rr / group_rows, gr = rr % group_rows;
  const size_t block = (size_t)tile_rows * kOzS * kOzBK;  // one K block of one tile
  const size_t slab = (size_t)group_rows * kOzBK;         // one digit of one group
  signed char* o = out + (size_t)tile * nkb * block + (size_t)grp * kOzS * slab;
  for (int k = threadIdx.x; k < nkb * kOzBK; k += blockDim.x) {
    double y = (live && k < K) ? ldexp(x[(long long)k * ld_k], 6 - e) : 0.0;  // |y| < 64
    signed char* ok = o + (size_t)(k / kOzBK) * block + oz_swz(gr, k % kOzBK);
#pragma unroll
    for (int t = 0; t < kOzS; ++t) {
      const double d = rint(y);
      ok[t * slab] = static_cast<signed char>(d);
      y = (y - d) * 128.0;  // exact: |y - d| <= 1/2
    }
  }
}

}  // namespace bnbg
