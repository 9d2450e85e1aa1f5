// Cell-update formulation microbenchmark for sm_100a (B200): can part of the
// s16x2 Gotoh cell update move off the ALU pipe?
//
// The pass kernel's cell pair costs 5.5 DPX on the ALU pipe (64 lane-ops/clk/SM,
// profiles/r01_dpx_microbench.jsonl) plus one IMAD (FMA pipe) that packs the
// two halves' profile scores.  fp16x2 adds (HADD2/HFMA2) issue on the FMA pipe.
// For values in [0, 2048] fp16 arithmetic on integers is exact, and for
// non-negative fp16 values the bit pattern orders like the value, so the s16x2
// integer max (VIMNMX/VIMNMX3) is an exact fp16 max whenever one operand is
// >= 0.  fp16 values in [1024, 2048) have ulp 1 and bits 0x6400 + (v - 1024):
// there an integer add on the bits IS the fp16 add, so DPX add-max and fp16
// adds can be mixed freely on "biased" values (v = 1024 + x).
//
// Variants (R rows x 1 column per step, 2 cells per register):
//   DPX  : the pass kernel's form (5.5 DPX + IMAD pack).
//   HA   : biased; t = HADD2(hd, sub); h = VIMNMX3(t, E, F);
//          hg = VIADDMNMX(h, -Goe, BIAS); E,F = VIADDMNMX(E/F, -Ge, hg)
//          (4.5 ALU + 2 FMA per pair-cell)
//   HB   : plain fp16; t = HADD2; h = VIMNMX3(t, E, F); u = HADD2(h, -Goe);
//          E = VIMNMX.RELU(HADD2(E, -Ge), u); F likewise
//          (3.5 ALU + 5 FMA per pair-cell)
//   HBF  : HB with hg = HFMA2.RELU(h, 1, -Goe) and plain VIMNMX for E/F
//   MIX  : biased, rows alternate HA / HB (max3 with BIAS) forms
//   *_I  : the -Goe/-Ge fp16 constants as compile-time immediates
// LDS=1 adds the pass kernel's profile traffic (two LDS.128 per 4 rows).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o hybrid_cell hybrid_cell.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 1024;
enum Var { DPX, HA, HB, HBF, MIX, HB_I, HBF_I, MIX_I, HA_I, HAINT, HAINT_T, HA_I_T, HC, HMIX2, HMIX3, SPV, HAI16, NUM_VARS };
static const char *kNames[] = {"dpx", "hybA_biased", "hybB_fp16", "hybB_fp16_fmarelu", "mix_AB_biased",
                               "hybB_fp16_imm", "hybB_fp16_fmarelu_imm", "mix_AB_biased_imm", "hybA_biased_imm", "hybA_int_imad", "hybA_int_imad_Stree", "hybA_biased_imm_Stree", "hybC_int_fmaroute", "hybAC_mix_1to1", "hybAC_mix_2to1", "score_profile_SP", "hybA_int_profile16"};

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ __half2 h2(uint32_t a) { return *reinterpret_cast<__half2 *>(&a); }
__device__ __forceinline__ uint32_t u32(__half2 a) { return *reinterpret_cast<uint32_t *>(&a); }
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) { return u32(__hadd2(h2(a), h2(b))); }
__device__ __forceinline__ uint32_t hadd2_m2(uint32_t a) {   // a + (-2.0, -2.0), immediate
  return u32(__hadd2(h2(a), __float2half2_rn(-2.0f)));
}
__device__ __forceinline__ uint32_t hadd2_m12(uint32_t a) {  // a + (-12.0, -12.0), immediate
  return u32(__hadd2(h2(a), __float2half2_rn(-12.0f)));
}
__device__ __forceinline__ uint32_t hfma2_relu(uint32_t a, uint32_t b, uint32_t c) {
  return u32(__hfma2_relu(h2(a), h2(b), h2(c)));
}
__device__ __forceinline__ uint32_t hfma2_relu_m12(uint32_t a) {  // relu(a*1 - 12), immediates
  return u32(__hfma2_relu(h2(a), __float2half2_rn(1.0f), __float2half2_rn(-12.0f)));
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int VAR, int R, bool LDS>
__global__ void __launch_bounds__(256, (R <= 8 ? 4 : 2)) bench(const uint32_t *__restrict__ in, uint32_t *out, long long *cycles, uint32_t one_p) {
  __shared__ uint4 prof[VAR == SPV ? 1 : 8 * (R / 4) * 32];
  for (int i = threadIdx.x; i < (VAR == SPV ? 1 : 8 * (R / 4) * 32); i += blockDim.x)
    prof[i] = make_uint4(in[i & 15], in[(i + 1) & 15], in[(i + 2) & 15], in[(i + 3) & 15]);
  const uint32_t ngoe = in[12], nge = in[13], bias = in[4], one = in[5];
  const uint32_t ngoe32 = in[8] * 0xfff4fff4u, nge32 = in[8] * 0xfffefffeu;
  const uint32_t ngoe_h = in[6], nge_h = in[7];
  uint32_t H[R], E[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { H[r] = in[r & 15] + threadIdx.x; E[r] = in[(r + 3) & 15]; }
  uint32_t S = 0, A0 = in[14], B0 = in[15], b = in[0], c = in[1];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(prof) + (threadIdx.x & 31) * 16;
  __shared__ uint32_t sptab[VAR == SPV ? 400 * 26 : 1];
  if (VAR == SPV)
    for (int i = threadIdx.x; i < 400 * 26; i += blockDim.x) sptab[i] = in[i & 15] * 0x10001u;
  const uint32_t spbase = (uint32_t)__cvta_generic_to_shared(sptab);
  uint32_t qoff[R];
#pragma unroll
  for (int r = 0; r < R; ++r) qoff[r] = ((threadIdx.x * 7 + r * 11) % 26) * 4;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    uint32_t F = b, hd = c;
    A0 += it;
    B0 ^= it;
    if constexpr (VAR == SPV) {
      // NEXT-1 score profile: the column's letter pair selects a
      // 26-word vector SP[c] = SM(c, dB) * 65536 + SM(c, dA) (built once per
      // matrix: a 26 x 26 x 26 table, no packing per cell); each row reads
      // SP[q_r] with its own query letter -> one LDS.32 per row, random banks.
      const uint32_t pairbase = spbase + (((it * 7) ^ (threadIdx.x * 13)) % 400) * 104;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t sub = lds32(pairbase + qoff[r]);
        uint32_t h = __vimax3_s16x2(imad(hd, one_p, sub), E[r], F);
        hd = H[r]; H[r] = h;
        const uint32_t hg = __viaddmax_s16x2(h, ngoe, 0x40004000u);
        E[r] = __viaddmax_s16x2(E[r], nge, hg);
        F = __viaddmax_s16x2(F, nge, hg);
      }
#pragma unroll
      for (int r = 0; r < R; r += 2) S = __vimax3_s16x2(S, H[r], H[r + 1]);
      b ^= F;
      c += S;
      continue;
    }
    if constexpr (VAR == HAI16) {
      // int16 query profile: one LDS.128 holds 8 rows of a letter (half the
      // shared-memory bytes of the 32-bit-word profile); the packed words are
      // rebuilt on the FMA pipe: 5 IMAD per 2 rows (+ the 2 diagonal adds)
      const uint32_t la16 = sbase + ((it * 7) & 7) * (R / 8) * 512;
      const uint32_t lb16 = sbase + ((it * 13) & 7) * (R / 8) * 512;
#pragma unroll
      for (int k = 0; k < R / 8; ++k) {
        const uint4 a4 = lds128(la16 + k * 512), b4 = lds128(lb16 + k * 512);
        const uint32_t aw[4] = {a4.x, a4.y, a4.z, a4.w}, bw[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t hiA = (uint32_t)__mulhi((int)aw[j], 65536);          // sext(a[r+1])
          const uint32_t loA = imad(hiA, 0xffff0000u, aw[j]);                 // sext(a[r])
          const uint32_t hiB = (uint32_t)__mulhi((int)bw[j], 65536);
          const uint32_t P0 = imad(bw[j], 65536u, loA), P1 = imad(hiB, 65536u, hiA);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = k * 8 + j * 2 + e;
            uint32_t h = __vimax3_s16x2(imad(hd, one_p, e ? P1 : P0), E[r], F);
            hd = H[r]; H[r] = h;
            const uint32_t hg = __viaddmax_s16x2(h, ngoe, 0x40004000u);
            E[r] = __viaddmax_s16x2(E[r], nge, hg);
            F = __viaddmax_s16x2(F, nge, hg);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; r += 2) S = __vimax3_s16x2(S, H[r], H[r + 1]);
      b ^= F;
      c += S;
      continue;
    }
    const uint32_t la = sbase + ((it * 7) & 7) * (R / 4) * 512;
    const uint32_t lb = sbase + ((it * 13) & 7) * (R / 4) * 512;
#pragma unroll
    for (int k = 0; k < R / 4; ++k) {
      uint4 a4, b4;
      if (LDS) { a4 = lds128(la + k * 512); b4 = lds128(lb + k * 512); }
      else { a4 = make_uint4(A0, A0 >> 1, A0 >> 2, A0 >> 3); b4 = make_uint4(B0, B0 >> 1, B0 >> 2, B0 >> 3); }
      const uint32_t av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = k * 4 + j;
        const uint32_t sub = imad(bv[j], 65536u, av[j]);
        uint32_t h;
        if (VAR == DPX) {
          h = __viaddmax_s16x2_relu(hd, sub, E[r]);
          h = __vmaxs2(h, F);
          hd = H[r]; H[r] = h;
          const uint32_t hg = __viaddmax_s16x2_relu(h, ngoe, ngoe);
          E[r] = __viaddmax_s16x2(E[r], nge, hg);
          F = __viaddmax_s16x2(F, nge, hg);
        } else if (VAR == HC || (VAR == HMIX2 && (r & 1)) || (VAR == HMIX3 && r % 3 == 2)) {
          // FMA route: u = h - Goe, e1 = E - Ge, f1 = F - Ge as 32-bit adds (no borrow:
          // values >= B = 16384 >= the clamped penalties); 3 max3 with the floor B
          h = __vimax3_s16x2(imad(hd, one_p, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t u = imad(h, one_p, ngoe32);
          E[r] = __vimax3_s16x2(imad(E[r], one_p, nge32), u, 0x40004000u);
          F = __vimax3_s16x2(imad(F, one_p, nge32), u, 0x40004000u);
        } else if (VAR == HAINT || VAR == HAINT_T || VAR == HMIX2 || VAR == HMIX3) {
          h = __vimax3_s16x2(imad(hd, one_p, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t hg = __viaddmax_s16x2(h, ngoe, 0x40004000u);
          E[r] = __viaddmax_s16x2(E[r], nge, hg);
          F = __viaddmax_s16x2(F, nge, hg);
        } else if (VAR == HA || VAR == HA_I || VAR == HA_I_T || ((VAR == MIX || VAR == MIX_I) && (r & 1) == 0)) {
          h = __vimax3_s16x2(hadd2(hd, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t hg = __viaddmax_s16x2(h, ngoe, (VAR == HA_I || VAR == HA_I_T) ? 0x64006400u : bias);
          E[r] = __viaddmax_s16x2(E[r], nge, hg);
          F = __viaddmax_s16x2(F, nge, hg);
        } else if (VAR == MIX || VAR == MIX_I) {
          h = __vimax3_s16x2(hadd2(hd, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t u = VAR == MIX_I ? hadd2_m12(h) : hadd2(h, ngoe_h);
          E[r] = __vimax3_s16x2(VAR == MIX_I ? hadd2_m2(E[r]) : hadd2(E[r], nge_h), u, bias);
          F = __vimax3_s16x2(VAR == MIX_I ? hadd2_m2(F) : hadd2(F, nge_h), u, bias);
        } else if (VAR == HB || VAR == HB_I) {
          h = __vimax3_s16x2(hadd2(hd, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t u = VAR == HB_I ? hadd2_m12(h) : hadd2(h, ngoe_h);
          E[r] = __vimax_s16x2_relu(VAR == HB_I ? hadd2_m2(E[r]) : hadd2(E[r], nge_h), u);
          F = __vimax_s16x2_relu(VAR == HB_I ? hadd2_m2(F) : hadd2(F, nge_h), u);
        } else {  // HBF, HBF_I
          h = __vimax3_s16x2(hadd2(hd, sub), E[r], F);
          hd = H[r]; H[r] = h;
          const uint32_t hg = VAR == HBF_I ? hfma2_relu_m12(h) : hfma2_relu(h, one, ngoe_h);
          E[r] = __vmaxs2(VAR == HBF_I ? hadd2_m2(E[r]) : hadd2(E[r], nge_h), hg);
          F = __vmaxs2(VAR == HBF_I ? hadd2_m2(F) : hadd2(F, nge_h), hg);
        }
      }
    }
    if (VAR == HAINT_T || VAR == HA_I_T) {   // S as a tree of VIMNMX3 (depth log3 R)
      uint32_t m[R];
      int n = R;
#pragma unroll
      for (int r = 0; r < R; ++r) m[r] = H[r];
#pragma unroll
      for (int lvl = 0; lvl < 6; ++lvl) {
        if (n > 1) {
          int k = 0;
#pragma unroll
          for (int i = 0; i + 2 < 32; i += 3) {
            if (i + 2 < n) m[k++] = __vimax3_s16x2(m[i], m[i + 1], m[i + 2]);
            else if (i + 1 < n) m[k++] = __vmaxs2(m[i], m[i + 1]);
            else if (i < n) m[k++] = m[i];
          }
          n = k;
        }
      }
      S = __vmaxs2(S, m[0]);
    } else {
#pragma unroll
    for (int r = 0; r < R; r += 2) S = __vimax3_s16x2(S, H[r], H[r + 1]);
    }
    b ^= F;
    c += S;
  }
  long long t1 = clock64();
  uint32_t acc = S;
#pragma unroll
  for (int r = 0; r < R; ++r) acc ^= H[r] ^ E[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}


enum PipeOp { P_HADD2_RR, P_HADD2_IMM, P_HMNMX2, P_MIX_DPX_HADD2_RR, P_MIX_DPX_HADD2_IMM, P_MIX_DPX_HMNMX2,
              P_MIX_DPX_HFMA2RELU_IMM, P_MIX_DPX2_HADD2IMM1, NUM_POPS };
static const char *kPNames[] = {"hadd2_rr", "hadd2_imm", "hmnmx2", "mix_dpx_hadd2_rr_1to1", "mix_dpx_hadd2_imm_1to1",
                                "mix_dpx_hmnmx2_1to1", "mix_dpx_hfma2relu_imm_1to1", "mix_dpx2_hadd2imm1"};
static const int kPOps[] = {1, 1, 1, 2, 2, 2, 2, 3};
template <int OP>
__global__ void __launch_bounds__(256) pbench(const uint32_t *__restrict__ in, uint32_t *out, long long *cycles) {
  constexpr int C = 8;
  uint32_t a[C];
  uint32_t c = in[1];
#pragma unroll
  for (int k = 0; k < C; ++k) a[k] = in[3 + k] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 2048; ++it) {
    uint32_t n[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const uint32_t x = a[k], y = a[(k + 1) % C];
      if (OP == P_HADD2_RR) n[k] = hadd2(x, y);
      else if (OP == P_HADD2_IMM) n[k] = hadd2_m2(x);
      else if (OP == P_HMNMX2) n[k] = u32(__hmax2(h2(x), h2(y)));
      else if (OP == P_MIX_DPX_HADD2_RR) n[k] = hadd2(__viaddmax_s16x2(x, y, c), y);
      else if (OP == P_MIX_DPX_HADD2_IMM) n[k] = hadd2_m2(__viaddmax_s16x2(x, y, c));
      else if (OP == P_MIX_DPX_HMNMX2) n[k] = u32(__hmax2(h2(__viaddmax_s16x2(x, y, c)), h2(y)));
      else if (OP == P_MIX_DPX_HFMA2RELU_IMM) n[k] = hfma2_relu_m12(__viaddmax_s16x2(x, y, c));
      else n[k] = hadd2_m2(__viaddmax_s16x2(__vimax3_s16x2(x, y, c), y, c));
    }
#pragma unroll
    for (int k = 0; k < C; ++k) a[k] = n[k];
    c += 0x10001u;
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) acc ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
template <int OP>
int prun(int nsm, int bps, uint32_t *d_in, uint32_t *d_out, long long *d_cyc) {
  const int threads = 256, blocks = nsm * bps;
  pbench<OP><<<blocks, threads>>>(d_in, d_out, d_cyc);
  CK(cudaDeviceSynchronize());
  pbench<OP><<<blocks, threads>>>(d_in, d_out, d_cyc);
  CK(cudaDeviceSynchronize());
  long long *h = new long long[blocks];
  CK(cudaMemcpy(h, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < blocks; ++i) if (h[i] > mx) mx = h[i];
  delete[] h;
  const double ops = 2048.0 * 8 * kPOps[OP] * threads * bps;
  printf("{\"pipe_op\": \"%s\", \"blocks_per_sm\": %d, \"thread_ops_per_clk_per_sm\": %.2f, \"warp_instr_per_clk_per_sm\": %.3f}\n",
         kPNames[OP], bps, ops / mx, ops / mx / 32);
  return 0;
}

template <int VAR, int R, bool LDS>
int run(int nsm, int bps, uint32_t *d_in, uint32_t *d_out, long long *d_cyc) {
  const int threads = 256, blocks = nsm * bps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench<VAR, R, LDS><<<blocks, threads>>>(d_in, d_out, d_cyc, 1u);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  bench<VAR, R, LDS><<<blocks, threads>>>(d_in, d_out, d_cyc, 1u);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long *h = new long long[blocks];
  CK(cudaMemcpy(h, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
  long long mx = 0; double mean = 0;
  for (int i = 0; i < blocks; ++i) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= blocks;
  delete[] h;
  const double cells = (double)ITERS * R * 2 * threads * bps;   // per SM
  printf("{\"var\": \"%s\", \"R\": %d, \"lds\": %d, \"blocks_per_sm\": %d, \"cells_per_clk_per_sm\": %.2f, "
         "\"max_block_cycles\": %lld, \"mean_block_cycles\": %.0f, \"ms\": %.3f, \"implied_sm_mhz\": %.0f}\n",
         kNames[VAR], R, (int)LDS, bps, cells / (double)mx, mx, mean, ms, (double)mx / (ms * 1e3));
  return 0;
}

template <int R, bool LDS>
void run_all(int nsm, uint32_t *d_in, uint32_t *d_out, long long *d_cyc, int bps = 2) {
  {
    run<DPX, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HA, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HB, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HBF, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HB_I, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HBF_I, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<MIX_I, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HA_I, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HAINT, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HAINT_T, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HA_I_T, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HC, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HMIX2, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<HMIX3, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    run<SPV, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
    if constexpr (R % 8 == 0) run<HAI16, R, LDS>(nsm, bps, d_in, d_out, d_cyc);
  }
}

int main() {
  int nsm = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint32_t h_in[16] = {0x00020003u, 0x00010001u, 0x5410u, 1, 0x64006400u, 0x3C003C00u, 0xCA00CA00u, 0xC000C000u,
                       8, 0, 0, 0, 0xfff4fff4u, 0xfffefffeu, 0x01020304u, 0x05060708u};
  uint32_t *d_in, *d_out; long long *d_cyc;
  CK(cudaMalloc(&d_in, sizeof(h_in)));
  CK(cudaMemcpy(d_in, h_in, sizeof(h_in), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_out, (size_t)nsm * 8 * 256 * sizeof(uint32_t)));
  CK(cudaMalloc(&d_cyc, (size_t)nsm * 8 * sizeof(long long)));
  printf("{\"device_sms\": %d}\n", nsm);
  for (int bps : {2, 4}) {
    prun<P_HADD2_RR>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_HADD2_IMM>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_HMNMX2>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_MIX_DPX_HADD2_RR>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_MIX_DPX_HADD2_IMM>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_MIX_DPX_HMNMX2>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_MIX_DPX_HFMA2RELU_IMM>(nsm, bps, d_in, d_out, d_cyc);
    prun<P_MIX_DPX2_HADD2IMM1>(nsm, bps, d_in, d_out, d_cyc);
  }
  run_all<8, true>(nsm, d_in, d_out, d_cyc, 4);
  run_all<16, true>(nsm, d_in, d_out, d_cyc, 2);
  run_all<28, true>(nsm, d_in, d_out, d_cyc, 2);
  return 0;
}
