// ozaki.cuh -- the expectation W = P V (Alg. 1 line 11; Markov form Eq. 6) on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM): SURVEY §8(f) NEXT-4, the
// "lower-precision path only if it meets the stated tolerance" of north_star.
//
// FP64 has no tcgen05 kind on sm_100a, so the FP64 product is emulated exactly in integers (the Ozaki
// scheme): every row m of P is scaled by 2^-e_m (e_m: the exponent just above the row's largest entry)
// and every column n of V by 2^-f_n, so the scaled entries lie in [0, 1); each is cut into kOzS = 8
// 8-bit digits, a = sum_p D_p 2^-8p + r with 0 <= r < 2^-64 (truncation; exact in FP64: one scaling by a
// power of two and one float->integer conversion).  Both operands are non-negative -- P is a stochastic
// matrix and V_{t+1} >= 0 (R18: the zero action is always feasible with payoff 0) -- so the digits are
// unsigned bytes.  Then
//     W[m][n] = 2^(e_m + f_n) sum_{p+q <= kOzS+1} 2^-8(p+q) (D^P_p D^V_q)[m][n]  +  truncation,
// where every D^P_p D^V_q is an exact u8 x u8 -> s32 tensor-core product.  The 36 products of the 8
// diagonals d = p + q - 2 accumulate in 8 TMEM accumulators (the tensor core adds them exactly in s32:
// K' <= 128 keeps every diagonal below 2^26), combined exactly in int64 and rounded once to FP64.
// Error per entry: <= 4 (2 K' 2^-64 + 64 2^-80) max_k' P[m][k'] max_k' V[k'][n] + one rounding -- pinned
// by tests/test_gpu_ozaki.py against an extended-precision product -- far inside north_star's 1e-9, but
// NOT the canonical fma chain of R15: W differs from the oracle's in the last bits, and a policy may
// differ where the oracle's top-2 candidates tie within that error (documented ties).
// Opt-in (ESDP_CONTRACT_OZAKI).
//
// One persistent CTA per SM, warp-specialized, 288 threads:
//   warps 0-3  digitizers: load a 64-column tile of V_{t+1} (FP64) in two halves of 32 columns (a warp reads
//              one row of the half per load), the column exponents (named barrier), and write the 8 digit
//              images of the tile into the digit-image slot (K-major UMMA layout);
//   warps 4-7  epilogue: tcgen05.ld the 8 accumulators of a tile, combine, scale, store W (FP64);
//   warp 8     TMEM allocation and the MMA issue (one lane: 36 digit products x 4 K-steps, straight-line).
// P's digit images (all of P_t: 128 rows x 128 k', 8 x 16 KB) are built once per CTA before the
// programmatic dependency wait (P is an input).  Shared memory: 128 KB of P images + one 64 KB V-image slot;
// TMEM: one accumulator set of 8 x 64 columns.  Digitizing tile j + 1 overlaps the epilogue of tile j.
//
// Measured on B200: correct, but SLOWER than the canonical FP64 DMMA expectation on the
// cfg5 batch GEMM ([100] x [128,512] per stage): 172 us (N = 64, this layout) and 173-179 us (N = 32 with two
// accumulator sets and a two-slot ring) vs 108 us per launch.  tools/microbench/mb10.cu: an M = 128, K = 32
// u8 MMA costs >= 46 cycles for any N <= 64 (shared-memory bound: the 4 KB A tile is re-read by every MMA)
// and reaches the 8.2K MAC/cycle peak only at N >= 128, but 8 accumulators x N TMEM columns <= 512 caps N
// at 64; with the 128 KB of P images resident, no shared memory is left to stage V tiles ahead, and ncu
// shows the digitizers waiting on their V loads and the epilogue on the MMAs.
#pragma once
#include "kernels.cuh"

namespace esdp {

constexpr int kOzS = 8;                       // 8-bit digits per operand (64 bits)
constexpr int kOzN = 64;                      // output columns per tile (UMMA N)
constexpr int kOzM = 128;                     // UMMA M: rows k of P, zero-padded
constexpr int kOzK = 128;                     // reduction k' zero-padded to 4 UMMA K-steps of 32 bytes
constexpr int kOzStages = 1;                  // digit-image slots (one: the A images take 128 KB)
constexpr int kOzAccCols = kOzS * kOzN;       // TMEM columns of the accumulator set (all 512)
constexpr int kOzThreads = 32 * 9;            // 4 digitizer, 4 epilogue, 1 MMA warp
constexpr int kOzImgA = kOzM * kOzK;          // bytes of one digit image of P (16 KB)
constexpr int kOzImgB = kOzN * kOzK;          // bytes of one digit image of a V tile (8 KB)
constexpr int kOzTileB = kOzS * kOzImgB;      // 64 KB
constexpr size_t kOzFixed = (size_t)kOzS * kOzImgA + (size_t)kOzStages * kOzTileB;
constexpr size_t kOzMisc = 6144;              // barriers (256 B), exponents (1 KB), column-maximum scratch (4 KB)
constexpr size_t kOzSmem = kOzFixed + kOzMisc;
static_assert(kOzS == 8, "the epilogue combines exactly 8 diagonal accumulators");
static_assert(kOzAccCols <= 512, "one accumulator set in TMEM");

// Byte (row r, k) of a K-major, SWIZZLE_NONE UMMA operand image: 8-row x 16-byte core matrices laid out
// [row group][k chunk][row in group][16 bytes]; next k chunk (LBO) 128 B, next row group (SBO) 1024 B.
__host__ __device__ constexpr int oz_off(int r, int k) { return (r >> 3) * 1024 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

// shared-memory matrix descriptor (tcgen05 "version 1"): start >> 4, LBO >> 4, SBO >> 4, no swizzle
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}
// instruction descriptor: s32 accumulator, unsigned 8-bit A and B, both K-major, N = 32, M = 128
constexpr uint32_t kOzIdesc = (2u << 4) | ((uint32_t)(kOzN >> 3) << 17) | ((uint32_t)(kOzM >> 4) << 24);

__device__ __forceinline__ void oz_mma(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kOzIdesc), "r"(acc));
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void oz_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void oz_fence_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void oz_bar_digitizers() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// TMEM lanes [32 (warp % 4), +32) x 8 consecutive 32-bit columns -> 8 registers of this lane's row
__device__ __forceinline__ void oz_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// exponent e with x < 2^e (x >= 0 finite); 0 for x == 0
__device__ __forceinline__ int oz_exp_above(double x) { return x > 0.0 ? ilogb(x) + 1 : 0; }
// 2^-e as a double (|e| <= 1022)
__device__ __forceinline__ double oz_pow2(int e) { return __longlong_as_double((long long)(1023 - e) << 52); }
// the 64 digit bits of a in [0, 1): trunc(a 2^64), exact
__device__ __forceinline__ unsigned long long oz_bits(double a) { return __double2ull_rz(a * 0x1p64); }
// digit p (1..8) of four values packed into one 32-bit word (byte j = value j)
__device__ __forceinline__ uint32_t oz_pack(unsigned long long x0, unsigned long long x1, unsigned long long x2,
                                            unsigned long long x3, int p) {
  const int sh = 64 - 8 * p;
  return (uint32_t)((x0 >> sh) & 255u) | ((uint32_t)((x1 >> sh) & 255u) << 8) | ((uint32_t)((x2 >> sh) & 255u) << 16) |
         ((uint32_t)((x3 >> sh) & 255u) << 24);
}
// the kOzS digit words of 16 consecutive k' of one row / column, written at byte offset off of each image
__device__ __forceinline__ void oz_digits16(const double (&v)[16], double sc, unsigned char* img, int img_bytes, int off) {
  unsigned long long x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = oz_bits(v[i] * sc);
#pragma unroll
  for (int p = 1; p <= kOzS; ++p) {
    uint4 w;
    w.x = oz_pack(x[0], x[1], x[2], x[3], p);
    w.y = oz_pack(x[4], x[5], x[6], x[7], p);
    w.z = oz_pack(x[8], x[9], x[10], x[11], p);
    w.w = oz_pack(x[12], x[13], x[14], x[15], p);
    *reinterpret_cast<uint4*>(img + (size_t)(p - 1) * img_bytes + off) = w;
  }
}

struct OzBars {
  uint64_t full, empty, tfull, tempty, fxready[2], fxfree[2];
  uint32_t taddr;
};

// W[m][n] (m < rows, n < ncols) = sum_k' P[m][k'] V[k'][n] with P [rows][K] (row stride K), V row stride ldv,
// W row stride ldw.  rows <= 128, K <= 128; entries of P and V non-negative and finite.
__global__ void __launch_bounds__(kOzThreads, 1) ozaki_contract_kernel(const double* __restrict__ Pt,
                                                                     const double* __restrict__ Vn,
                                                                     double* __restrict__ Wt, int rows, int K,
                                                                     long long ncols, long long ldv, long long ldw) {
  extern __shared__ __align__(16) unsigned char ozsm[];   // no-swizzle operand images need 16-byte alignment only
  unsigned char* imgA = ozsm;                                         // [kOzS][kOzImgA]
  unsigned char* imgB = imgA + (size_t)kOzS * kOzImgA;                // [kOzStages][kOzS][kOzImgB]
  OzBars* bars = reinterpret_cast<OzBars*>(imgB + (size_t)kOzStages * kOzTileB);
  int* eexp = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(bars) + 256);   // [128] row exponents
  int* fexp = eexp + 128;                                                              // [2][kOzN] column exponents
  double* cmax = reinterpret_cast<double*>(fexp + 2 * kOzN);                           // [2][4][kOzN] partial maxima
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long ntiles = (ncols + kOzN - 1) / kOzN;
  ESDP_ASSERT(blockDim.x == kOzThreads && rows <= kOzM && K <= kOzK && rows >= 1 && K >= 1);

  if (tid == 0) {
    mbar_init(&bars->full, 128); mbar_init(&bars->empty, 1);
    mbar_init(&bars->tfull, 1); mbar_init(&bars->tempty, 128);
    for (int b = 0; b < 2; ++b) { mbar_init(&bars->fxready[b], 128); mbar_init(&bars->fxfree[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {   // TMEM: the accumulator set (8 x 64 = 512 columns); one CTA per SM (shared memory)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&bars->taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // digit images of P (an input: before the dependency wait).  Item (row r, 16-k' chunk c): 8 consecutive
  // threads hold one row, so the row maximum is a 3-step shuffle.
  for (int it0 = 0; it0 < kOzM * 8; it0 += kOzThreads) {
    const int item = it0 + tid, r = item >> 3, c = item & 7;
    const bool live = item < kOzM * 8 && r < rows;
    double v[16];
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = 16 * c + i;
      v[i] = (live && k < K) ? __ldg(Pt + (size_t)r * K + k) : 0.0;
      mx = fmax(mx, v[i]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = oz_exp_above(mx);
    if (item < kOzM * 8) {
      if (c == 0) eexp[r] = e;
      oz_digits16(v, oz_pow2(e), imgA, kOzImgA, oz_off(r, 16 * c));
    }
  }
  oz_fence_proxy();          // generic-proxy stores of the P images -> visible to the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars->taddr;
  pdl_wait();                // V_{t+1} is the previous kernel's output

  // Pipeline per tile `it` (one digit-image slot, one TMEM accumulator set; phases stay within one of their
  // waiters, see the waits):  digitize(it) after MMA(it - 1) read the slot and the epilogue of it - 2 read
  // fexp[it & 1];  MMA(it) after digitize(it) and the epilogue of it - 1 drained TMEM;  epilogue(it) after
  // MMA(it) and digitize(it)'s column exponents.  Digitize(it + 1) overlaps epilogue(it).
  if (warp < 4) {
    // ---------------- digitizers: columns in two halves of 32; thread (column lane, k' part h = warp):
    // chunks h and h + 4 of 16 k' each; a warp reads one row of the half tile (32 doubles) per load
    const int h = warp;
    long long it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = (int)(it & 1);
      mbar_wait(&bars->empty, (unsigned)((it & 1) ^ 1));                  // the slot: MMAs of it - 1 done
      mbar_wait(&bars->fxfree[b], (unsigned)(((it >> 1) & 1) ^ 1));       // fexp[b]: epilogue of it - 2 done
      double* cm = cmax + (size_t)b * 4 * kOzN;
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        const int r = 32 * hh + lane;
        const long long n = tile * kOzN + r;
        const bool col = n < ncols;
        double v[2][16];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int k = 16 * (h + 4 * j) + i;
            v[j][i] = (col && k < K) ? __ldcg(Vn + (size_t)k * ldv + n) : 0.0;
          }
        double mx = 0.0;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 16; ++i) mx = fmax(mx, v[j][i]);
        cm[h * kOzN + r] = mx;
        oz_bar_digitizers();
        mx = fmax(fmax(cm[r], cm[kOzN + r]), fmax(cm[2 * kOzN + r], cm[3 * kOzN + r]));
        const int f = oz_exp_above(mx);
        if (h == 0) fexp[b * kOzN + r] = f;
        const double sc = oz_pow2(f);
#pragma unroll
        for (int j = 0; j < 2; ++j) oz_digits16(v[j], sc, imgB, kOzImgB, oz_off(r, 16 * (h + 4 * j)));
      }
      oz_fence_proxy();
      oz_arrive(&bars->full);
      oz_arrive(&bars->fxready[b]);
    }
  } else if (warp < 8) {
    // ---------------- epilogue: this warp's TMEM lanes = rows 32 (warp % 4) .. + 31
    const int m = 32 * (warp & 3) + lane;
    const uint32_t lanebase = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    const int e = eexp[m];
    long long it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = (int)(it & 1);
      mbar_wait(&bars->fxready[b], (unsigned)((it >> 1) & 1));   // the column exponents of tile it
      mbar_wait(&bars->tfull, (unsigned)(it & 1));
      tc_fence_after();
      const long long n0 = tile * kOzN;
#pragma unroll 1
      for (int cc = 0; cc < kOzN / 8; ++cc) {
        uint32_t acc[kOzS][8];
#pragma unroll
        for (int d = 0; d < kOzS; ++d) oz_ld8(lanebase + (uint32_t)(d * kOzN + cc * 8), acc[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        double out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          // exact: hi = sum_{d<4} acc_d 2^8(3-d) < 2^51, lo = sum_{d>=4} acc_d 2^8(7-d) < 2^51 (acc_d < 2^26)
          unsigned long long hi = acc[0][j];
          hi = (hi << 8) + acc[1][j];
          hi = (hi << 8) + acc[2][j];
          hi = (hi << 8) + acc[3][j];
          unsigned long long lo = acc[4][j];
          lo = (lo << 8) + acc[5][j];
          lo = (lo << 8) + acc[6][j];
          lo = (lo << 8) + acc[7][j];
          // sum_d acc_d 2^-8(d+2) = hi 2^-40 + lo 2^-72, rounded once; then the exact power-of-two scale
          const double sum = __fma_rn((double)hi, 0x1p-40, (double)lo * 0x1p-72);
          out[j] = sum * oz_pow2(-(e + fexp[b * kOzN + cc * 8 + j]));
        }
        if (m < rows) {
          double* wr = Wt + (size_t)m * ldw + n0 + cc * 8;
          if (n0 + cc * 8 + 8 <= ncols && ((reinterpret_cast<uintptr_t>(wr) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 8; j += 2) __stcg(reinterpret_cast<double2*>(wr + j), make_double2(out[j], out[j + 1]));  // stays in L2 for the stencil
          } else {
            for (int j = 0; j < 8; ++j)
              if (n0 + cc * 8 + j < ncols) wr[j] = out[j];
          }
        }
      }
      tc_fence_before();
      oz_arrive(&bars->tempty);
      oz_arrive(&bars->fxfree[b]);
    }
  } else {
    // ---------------- MMA issue (warp 8, one lane).  A descriptor's start-address field is (address >> 4) in
    // the low 14 bits and shared addresses stay below 2^18, so an operand at byte offset o is the base
    // descriptor plus o >> 4: the 144 MMAs of a tile are straight-line code with immediate offsets.
    long long it = 0;
    const uint64_t adesc = oz_desc(smem_u32(imgA)), bdesc = oz_desc(smem_u32(imgB));
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      mbar_wait(&bars->full, (unsigned)(it & 1));
      mbar_wait(&bars->tempty, (unsigned)((it & 1) ^ 1));   // the epilogue of it - 1 drained TMEM
      tc_fence_after();
      if (lane == 0) {
        // digit products D^P_(p+1) D^V_(q+1) with p + q <= kOzS - 1, into accumulator d = p + q.  K-steps
        // outermost, so consecutive MMAs update different accumulators; the first product of each diagonal
        // (first K-step, q = 0) overwrites it.
#pragma unroll
        for (int ks = 0; ks < kOzK / 32; ++ks)
#pragma unroll
          for (int q = 0; q < kOzS; ++q)
#pragma unroll
            for (int p = 0; p + q < kOzS; ++p)
              oz_mma(tbase + (uint32_t)((p + q) * kOzN), adesc + (uint64_t)((p * kOzImgA + ks * 256) >> 4),
                     bdesc + (uint64_t)((q * kOzImgB + ks * 256) >> 4), (q > 0 || ks > 0) ? 1u : 0u);
        oz_commit(&bars->empty);   // the slot is free once these MMAs have read it
        oz_commit(&bars->tfull);   // the accumulators of tile it are complete
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
  }
  pdl_trigger_late();
}

}  // namespace esdp
