// DPX / integer-pipe issue-rate microbenchmark for sm_100a (B200).
//
// Purpose: the cell-update roofline
// of the inter-task Smith-Waterman kernel is the per-SM issue rate of the pipe
// that the DPX instructions (VIADDMNMX.S16x2, VIMNMX.S16x2, VIMNMX3.S16x2) go
// to, divided by the instructions per cell.  MEASURED_PEAKS.json has no integer
// peak, so it is measured here: thread-ops per SM per clock for each op class
// alone and in 1:1 mixes (a mix that runs at the sum of the two rates proves
// the two classes issue to different pipes).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o dpx_microbench dpx_microbench.cu
// Output: one JSON line per op class on stdout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CHAINS = 8;
constexpr int ITERS = 2048;

enum Op { ADDMAX_RELU, ADDMAX, MAX2, MAX3, ADDMAX_S32, PRMT_OP, IADD3_OP, LOP3_OP, IMAD_OP,
          MIX_DPX_PRMT, MIX_DPX_IMAD, MIX_DPX_IADD3, CELL, SHFL_OP,
          MIX_DPX3_IMAD1, MIX_DPX_IMADIMM, MIX_DPX_IMADHALF, ADDMAX_RZ, MIX_DPX_MOV, CELL_U8X4,
          CELL_S16X2_EMU, NUM_OPS };
static const char* kNames[] = {"viaddmax_s16x2_relu", "viaddmax_s16x2", "vmax_s16x2", "vimax3_s16x2",
  "viaddmax_s32_relu", "prmt", "iadd3", "lop3", "imad", "mix_dpx_prmt_1to1", "mix_dpx_imad_1to1",
  "mix_dpx_iadd3_1to1", "cellpair_R8", "shfl_up", "mix_dpx3_imad1", "mix_dpx_imad_imm_1to1",
  "mix_dpx2_imad1", "viaddmax_relu_rz", "mix_dpx_mov_1to1", "cell_u8x4_R8", "cell_s16x2_sat_emul_R8"};
// thread-ops counted per chain per iteration for each op
static const int kOpsPerIter[] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 0, 2, 4, 2, 3, 1, 2, 0, 0};

template <int OP>
__global__ void __launch_bounds__(256) bench(const unsigned* __restrict__ in, unsigned* out,
                                             long long* cycles) {
  unsigned b = in[0], c = in[1], sel = in[2];
  unsigned a[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) a[k] = in[3 + k] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  if constexpr (OP == CELL) {
    // 8 query rows x 1 DB column of the s16x2 Gotoh update, as in the kernel.
    unsigned H[8], E[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) { H[r] = a[r]; E[r] = a[r] ^ b; }
    unsigned S = 0, zero = in[11], ngoe = in[12], nge = in[13];
    unsigned A0 = in[14], B0 = in[15];
    for (int it = 0; it < ITERS; ++it) {
      unsigned F = b, hd = c;
      A0 += it; B0 ^= it;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        unsigned sub = __byte_perm(A0, B0, 0x5410 + r);
        unsigned h = __viaddmax_s16x2_relu(hd, sub, E[r]);
        h = __vmaxs2(h, F);
        hd = H[r];
        H[r] = h;
        unsigned hg = __viaddmax_s16x2_relu(h, ngoe, zero);
        E[r] = __viaddmax_s16x2(E[r], nge, hg);
        F = __viaddmax_s16x2(F, nge, hg);
      }
#pragma unroll
      for (int r = 0; r < 8; r += 2) S = __vimax3_s16x2(S, H[r], H[r + 1]);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = H[r] ^ E[r];
    a[0] ^= S;
  } else if constexpr (OP == CELL_U8X4) {
    // NEXT-4: the paper's 8-bit lanes as 4 x u8 per register,
    // biased unsigned saturating arithmetic (SWIPE/Farrar style):
    //   h = subs(adds(hd, sub+bias), bias); h = max(h, E, F); S = max(S, h)
    //   hg = subs(h, Goe); E = max(subs(E, Ge), hg); F = max(subs(F, Ge), hg)
    // No DPX form exists for 8-bit lanes: __vaddus4 / __vsubus4 / __vmaxu4 are
    // multi-instruction emulations.  8 rows x 1 column x 4 lanes per iteration.
    unsigned H[8], E[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) { H[r] = a[r]; E[r] = a[r] ^ b; }
    unsigned S = 0, bias = in[11] | 0x04040404u, goe = 0x0c0c0c0cu, ge = 0x02020202u;
    unsigned A0 = in[14], B0 = in[15];
    for (int it = 0; it < ITERS; ++it) {
      unsigned F = b, hd = c;
      A0 += it; B0 ^= it;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        unsigned sub = __byte_perm(A0, B0, 0x5410 + r);
        unsigned h = __vsubus4(__vaddus4(hd, sub), bias);
        h = __vmaxu4(__vmaxu4(h, E[r]), F);
        hd = H[r];
        H[r] = h;
        S = __vmaxu4(S, h);
        unsigned hg = __vsubus4(h, goe);
        E[r] = __vmaxu4(__vsubus4(E[r], ge), hg);
        F = __vmaxu4(__vsubus4(F, ge), hg);
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = H[r] ^ E[r];
    a[0] ^= S;
  } else if constexpr (OP == CELL_S16X2_EMU) {
    // 16-bit lanes with the paper's *saturating* adds (__vaddss2 emulation)
    // instead of wrapping DPX: same recurrence, 8 rows x 2 lanes per iteration.
    unsigned H[8], E[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) { H[r] = a[r]; E[r] = a[r] ^ b; }
    unsigned S = 0, ngoe = in[12], nge = in[13];
    unsigned A0 = in[14], B0 = in[15];
    for (int it = 0; it < ITERS; ++it) {
      unsigned F = b, hd = c;
      A0 += it; B0 ^= it;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        unsigned sub = __byte_perm(A0, B0, 0x5410 + r);
        unsigned h = __vmaxs2(__vmaxs2(__vaddss2(hd, sub), E[r]), F);
        h = __vmaxs2(h, 0u);
        hd = H[r];
        H[r] = h;
        S = __vmaxs2(S, h);
        unsigned hg = __vmaxs2(__vaddss2(h, ngoe), 0u);
        E[r] = __vmaxs2(__vaddss2(E[r], nge), hg);
        F = __vmaxs2(__vaddss2(F, nge), hg);
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = H[r] ^ E[r];
    a[0] ^= S;
  } else {
    for (int it = 0; it < ITERS; ++it) {
      unsigned n[CHAINS];
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) {
        const unsigned x = a[k], y = a[(k + 1) % CHAINS];
        if constexpr (OP == ADDMAX_RELU) n[k] = __viaddmax_s16x2_relu(x, y, c);
        else if constexpr (OP == ADDMAX) n[k] = __viaddmax_s16x2(x, y, c);
        else if constexpr (OP == MAX2) n[k] = __vmaxs2(x, y) + 0;
        else if constexpr (OP == MAX3) n[k] = __vimax3_s16x2(x, y, c);
        else if constexpr (OP == ADDMAX_S32) n[k] = (unsigned)__viaddmax_s32_relu((int)x, (int)y, (int)c);
        else if constexpr (OP == PRMT_OP) n[k] = __byte_perm(x, y, sel);
        else if constexpr (OP == IADD3_OP) n[k] = x + y + c;
        else if constexpr (OP == LOP3_OP) n[k] = (x & y) ^ c;
        else if constexpr (OP == IMAD_OP) n[k] = x * y + c;
        else if constexpr (OP == MIX_DPX_PRMT) n[k] = __byte_perm(__viaddmax_s16x2(x, y, c), y, sel);
        else if constexpr (OP == MIX_DPX_IMAD) n[k] = __viaddmax_s16x2(x, y, c) * y + c;
        else if constexpr (OP == MIX_DPX_IADD3) n[k] = __viaddmax_s16x2(x, y, c) + y + b;
        else if constexpr (OP == SHFL_OP) n[k] = __shfl_up_sync(0xffffffffu, x, 1) ^ y;
        else if constexpr (OP == MIX_DPX3_IMAD1) {
          uint32_t t1 = __viaddmax_s16x2(x, y, c);
          uint32_t t2 = __viaddmax_s16x2_relu(t1, b, y);
          uint32_t t3 = __vimax3_s16x2(t2, x, c);
          uint32_t m;
          asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(m) : "r"(t3), "r"(y), "r"(b));
          n[k] = m;
        }
        else if constexpr (OP == MIX_DPX_IMADIMM) {
          uint32_t m;
          asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(m) : "r"(__viaddmax_s16x2(x, y, c)), "r"(y));
          n[k] = m;
        }
        else if constexpr (OP == MIX_DPX_IMADHALF) {
          uint32_t t1 = __viaddmax_s16x2(x, y, c);
          uint32_t t2 = __viaddmax_s16x2_relu(t1, b, y);
          uint32_t m;
          asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(m) : "r"(t2), "r"(x));
          n[k] = m;
        }
        else if constexpr (OP == ADDMAX_RZ) n[k] = __viaddmax_s16x2_relu(x, y, 0u);
        else if constexpr (OP == MIX_DPX_MOV) {
          uint32_t m;
          asm volatile("mov.b32 %0, %1;" : "=r"(m) : "r"(__viaddmax_s16x2(x, y, c)));
          n[k] = m;
        }
      }
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) a[k] = n[k];
      c += sel;
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) acc ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
int run(int nsm, int blocks_per_sm, unsigned* d_in, unsigned* d_out, long long* d_cyc) {
  const int threads = 256, blocks = nsm * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench<OP><<<blocks, threads>>>(d_in, d_out, d_cyc);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  bench<OP><<<blocks, threads>>>(d_in, d_out, d_cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  CK(cudaMemcpy(h, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
  double mean = 0; long long mx = 0;
  for (int i = 0; i < blocks; ++i) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= blocks;
  delete[] h;
  double ops_per_thread;
  if (OP == CELL) ops_per_thread = (double)ITERS * (8 * 5 + 8 /*prmt*/ + 4 /*max3*/);  // 5 DPX + 1 PRMT per row, 0.5 VIMNMX3
  else if (OP == CELL_U8X4) ops_per_thread = (double)ITERS * 8 * 4;       // CELLS (4 lanes x 8 rows)
  else if (OP == CELL_S16X2_EMU) ops_per_thread = (double)ITERS * 8 * 2;  // CELLS (2 lanes x 8 rows)
  else ops_per_thread = (double)ITERS * CHAINS * kOpsPerIter[OP];
  double ops_per_sm = ops_per_thread * threads * blocks_per_sm;
  double per_clk = ops_per_sm / (double)mx;          // thread-ops / clk / SM (all blocks concurrent)
  double eff_mhz = (double)mx / (ms * 1e3);          // cycles per microsecond of wall time
  printf("{\"op\": \"%s\", \"blocks_per_sm\": %d, \"threads\": %d, \"thread_ops_per_clk_per_sm\": %.2f, "
         "\"warp_instr_per_clk_per_sm\": %.3f, \"mean_block_cycles\": %.0f, \"max_block_cycles\": %lld, "
         "\"ms\": %.3f, \"implied_sm_mhz\": %.0f}\n",
         kNames[OP], blocks_per_sm, threads, per_clk, per_clk / 32.0, mean, mx, ms, eff_mhz);
  return 0;
}

int main() {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  unsigned h_in[16] = {0x00020003u, 0x00010001u, 0x5410u, 1, 2, 3, 4, 5, 6, 7, 8, 0, 0xfff4fff4u,
                       0xfffefffeu, 0x01020304u, 0x05060708u};
  unsigned* d_in; unsigned* d_out; long long* d_cyc;
  CK(cudaMalloc(&d_in, sizeof(h_in)));
  CK(cudaMemcpy(d_in, h_in, sizeof(h_in), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_out, (size_t)nsm * 8 * 256 * sizeof(unsigned)));
  CK(cudaMalloc(&d_cyc, (size_t)nsm * 8 * sizeof(long long)));
  printf("{\"device_sms\": %d}\n", nsm);
  for (int bps : {2, 4}) {
    run<ADDMAX_RELU>(nsm, bps, d_in, d_out, d_cyc);
    run<ADDMAX>(nsm, bps, d_in, d_out, d_cyc);
    run<MAX2>(nsm, bps, d_in, d_out, d_cyc);
    run<MAX3>(nsm, bps, d_in, d_out, d_cyc);
    run<ADDMAX_S32>(nsm, bps, d_in, d_out, d_cyc);
    run<PRMT_OP>(nsm, bps, d_in, d_out, d_cyc);
    run<IADD3_OP>(nsm, bps, d_in, d_out, d_cyc);
    run<LOP3_OP>(nsm, bps, d_in, d_out, d_cyc);
    run<IMAD_OP>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_PRMT>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_IMAD>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_IADD3>(nsm, bps, d_in, d_out, d_cyc);
    run<CELL>(nsm, bps, d_in, d_out, d_cyc);
    run<SHFL_OP>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX3_IMAD1>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_IMADIMM>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_IMADHALF>(nsm, bps, d_in, d_out, d_cyc);
    run<ADDMAX_RZ>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_DPX_MOV>(nsm, bps, d_in, d_out, d_cyc);
    run<CELL_U8X4>(nsm, bps, d_in, d_out, d_cyc);
    run<CELL_S16X2_EMU>(nsm, bps, d_in, d_out, d_cyc);
  }
  return 0;
}
