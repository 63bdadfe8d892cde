// gemm.cu — BF16 mode: the two big "all vertices at once" contractions of a pass, as row-tiled
// tcgen05 GEMMs (M = 128 position rows per CTA, N = BN weight rows, K-major operands via TMA,
// fp32 accumulators in TMEM), each with the cell epilogue fused (cells.cuh):
//   * eager pull projection (§3.5 "eager"): Z = X W^T over the pulled rows;
//     level-0 vertices finish the whole cell F here, x-vertices above level 0 keep Z (XW);
//   * pull's adjoint dX = dZ W (lazily batched) for the rows with a pull record.
// Unlike the level kernels the row count here is large (every vertex with a pull record), so
// the tile is the plain GEMM orientation: one thread per position row in the epilogue (TMEM
// lane = row), BN columns per CTA; for the Tree-LSTM x-projection the BN = 4 x 32 columns are
// the i, o, u, f rows of the same 32 units (B loaded as 4 boxes), so a thread owns all gates
// of its (vertex, unit) pairs.
//   warp 0: TMA producer, warp 1: TMEM allocator + MMA issuer, warps 2-5: epilogue.
// Rows tiles without any row needing the epilogue (no level-0 vertex and no pull record) exit
// at once (k_pull's per-64-row flags).
#include <cudaTypedefs.h>

#include <algorithm>

#include "cells.cuh"
#include "gemm.h"
#include "ptx.cuh"

namespace cavs {

constexpr int kGThreads = 192;
constexpr int kGRows = 128;            // position rows per CTA (MMA M)
constexpr int kGA = kGRows * 128;      // A stage: 128 rows x 64 k (bf16) = 16 KB

// mbarrier wait (try_wait, hardware-suspended), trapping after ~4 s instead of hanging
__device__ __forceinline__ void pwait_g(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  unsigned long long t0 = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    const unsigned long long now = gtime();
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
  }
}

__device__ __forceinline__ uint64_t g_desc(uint32_t saddr) {
  return ((uint64_t)((1024u >> 4) | (1u << 14) | (2u << 29)) << 32) | (((saddr >> 4) & 0x3FFF) | (1u << 16));
}

// E: epilogue kind; BN: accumulator columns; NG: row groups of B (gates) -> UGN = BN / NG units.
template <int E, int BN, int NG, int S>
__global__ void __launch_bounds__(kGThreads, 1)
k_gemm_rows(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, Dev D, int K,
            int a_col0, int b_gate_stride, int units) {
  constexpr int UGN = BN / NG;
  constexpr int BST = BN * 128;                          // B stage bytes
  constexpr int STAGE = kGA + BST;
  extern __shared__ __align__(16) uint8_t g_raw[];
  uint8_t* smem = g_raw + ((1024u - (ptx::smem_u32(g_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = blockIdx.x * kGRows;
  const int u0 = blockIdx.y * UGN;
  ptx::griddep_wait();                                   // flags / arenas of the previous kernels
  // PDL: the next kernel (the persistent forward after the x-projection) may launch once every CTA
  // of this grid is resident, so its prologue (weights -> TMEM) overlaps this grid's last wave; its
  // own griddepcontrol.wait still orders every read of this grid's outputs
  if (threadIdx.x == 0) ptx::griddep_launch();
  if (dev_skip(D)) return;                               // sync-free mode: invalid / DAG batch
  // rows needing the epilogue: level-0 vertices (x-projection) or pull records (k_pull's flags)
  {
    const int f0 = p0 >> 6;
    bool act = D.tile_x[f0] || (p0 + 64 < D.V && D.tile_x[f0 + 1]);
    if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ) act = act || p0 < dev_lp1(D);
    if (!act || p0 >= D.V) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = K / 64;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch(&mA); ptx::tma_prefetch(&mB);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        if (kb >= S) pwait_g(&empty[s], ((kb / S) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE;
        ptx::mbar_arrive_expect_tx(&full[s], STAGE);
        if constexpr (NG > 1)                            // all NG gate-row groups in ONE 4-D box (r02):
          ptx::tma_load_4d(st + kGA, &mB, 0, u0, kb, 0, &full[s]);   // an SM's boxes are serviced serially
        else
          ptx::tma_load_2d(st + kGA, &mB, kb * 64, u0, &full[s]);
        ptx::tma_load_2d(st, &mA, a_col0 + kb * 64, p0, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(kGRows, BN, 0, 0);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        pwait_g(&full[s], (kb / S) & 1);
        ptx::tc_fence_after();
        const uint32_t a = ptx::smem_u32(smem + s * STAGE), b = a + kGA;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16(tmem, g_desc(a + kk * 32), g_desc(b + kk * 32), idesc, (kb | kk) ? 1u : 0u);
        ptx::mma_commit(&empty[s]);
      }
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else {
    // ---- epilogue.  (1) thread = position row (TMEM lane): accumulators -> smem xs[row][col]
    //      (the pipeline buffers are free once `done` fired) + the row's metadata;
    //      (2) thread -> (row, 4-unit quad), quads of a row on consecutive lanes, so every store
    //      of the cell epilogue is a coalesced run of the row ----
    constexpr int PITCH = BN + 4;                        // floats; float4 rows conflict-free
    constexpr int QU = UGN / 4;                          // unit quads per row
    float* xs = reinterpret_cast<float*>(smem);
    VMeta* s_meta = reinterpret_cast<VMeta*>(smem + kGRows * PITCH * 4);
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 64;                     // 0..127
    {
      const int p = p0 + row;
      pwait_g(done, 0);
      ptx::tc_fence_after();
      const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        ptx::tmem_ld16(tq + c0, v);
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(xs + row * PITCH + c0 + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
      VMeta m;
      m.p = -1;
      if (p < D.V && row_active<E>(D, p, D.xrow_pos[p])) load_meta(D, p, false, m);
      s_meta[row] = m;
    }
    ptx::named_bar_sync(1, 128);
    const int uq = et % QU;
    const int j = u0 + uq * 4;
    if (j < units) {
      const UnitC<4> uc = epi_uses_bias<E>() ? load_unit<4>(D, j, epi_is_lstm<E>()) : UnitC<4>{};
#pragma unroll 1
      for (int r = et / QU; r < kGRows; r += 128 / QU) {
        const VMeta& m = s_meta[r];
        if (m.p < 0) continue;
        FV<4> acc[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const float4 x = *reinterpret_cast<const float4*>(xs + r * PITCH + g * UGN + uq * 4);
          acc[g].v[0] = x.x; acc[g].v[1] = x.y; acc[g].v[2] = x.z; acc[g].v[3] = x.w;
        }
        typename EpiK<E>::template In<4, 1> in;
        EpiK<E>::template load<4, 1>(D, j, m, in);
        EpiK<E>::template store<__nv_bfloat16, 4, 1>(D, j, m, acc, in, uc);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem);
  }
}

// =====================================================================================
struct GemmState {
  CUtensorMap A_xp, A_dz;       // arena rows, box {64, 128}
  CUtensorMap B_xp, B_dx;       // weight rows: x-projection (Tree-LSTM: 4-D, all gates in one box), dX
  bool ok = false;
};

static PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

// [NG x rows x K] weight rows viewed as {64 k, rows, k-block, gate}: box {64, box_rows, 1, NG} = the NG gate
// groups of box_rows rows of one k-block, smem order [gate][row][64] (the B tile of NG x box_rows rows)
static bool genc4(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint32_t ng, uint32_t box_rows) {
  cuuint64_t dims[4] = {64, rows, K / 64, ng};
  cuuint64_t strides[3] = {K * 2, 128, rows * K * 2};
  cuuint32_t box[4] = {64, box_rows, 1, ng};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool genc(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tree-LSTM x-projection: BN = 128 = 4 gates x 32 units; Tree-FC: BN = 128 units; dX: BN = 128.
constexpr int kXpBN = 128;
constexpr int kDxBN = 128;
constexpr int kGS = 3;                                     // pipeline stages (32 KB each): 2 CTAs per SM

template <int E, int BN, int NG>
static void launch_rows(const CUtensorMap& a, const CUtensorMap& b, const Dev& D, int K, int a_col0, int gate_stride,
                        int units, cudaStream_t s) {
  constexpr int smem = 1024 + kGS * (kGA + BN * 128) + 2 * kGS * 8 + 64;
  static_assert(kGRows * (BN + 4) * 4 + kGRows * (int)sizeof(VMeta) <= kGS * (kGA + BN * 128), "epilogue staging");
  static bool attr[kMaxDev] = {};
  const int dv = cur_device();
  if (!attr[dv]) {
    cudaFuncSetAttribute(k_gemm_rows<E, BN, NG, kGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[dv] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cdiv(D.V, kGRows), cdiv(units, BN / NG), 1);
  cfg.blockDim = dim3(kGThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_gemm_rows<E, BN, NG, kGS>, a, b, D, K, a_col0, gate_stride, units);
}

GemmState* gemm_init(const Dev& D, int max_vertices) {
  const char* env = std::getenv("CAVS_GEMM_ROWS");
  if (env && env[0] == '0') return nullptr;
  if (!g_enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return nullptr;
    g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const uint64_t h = D.h, d = D.d, Vp = (uint64_t)max_vertices + kPadRows;
  const uint64_t G = lstm ? 3 + D.N : 1;
  if (h % 32 || d % 128 || h % 128) return nullptr;
  GemmState* g = new GemmState();
  bool ok = genc(&g->A_xp, D.Xp, d, Vp, kGRows) && genc(&g->A_dz, D.dZ, G * h, Vp, kGRows);
  if (lstm) ok = ok && genc4(&g->B_xp, D.Wb, d, h, 4, kXpBN / 4);    // W4 [4h x d]: gate rows g*h + u
  else ok = ok && genc(&g->B_xp, D.Wb, d, h, kXpBN);                  // W_x [h x d]
  ok = ok && genc(&g->B_dx, D.We, G * h, d, kDxBN);                   // W^T [d x G h]
  if (!ok) { delete g; return nullptr; }
  g->ok = true;
  return g;
}

void gemm_destroy(GemmState* g) { delete g; }

bool gemm_xproj(const Dev& D, GemmState* g, cudaStream_t s) {
  if (!g) return false;
  if (D.cell == CAVS_CELL_TREE_LSTM)
    launch_rows<EPI_LSTM_XPROJ, kXpBN, 4>(g->A_xp, g->B_xp, D, D.d, 0, D.h, D.h, s);
  else
    launch_rows<EPI_FC_XPROJ, kXpBN, 1>(g->A_xp, g->B_xp, D, D.d, 0, 0, D.h, s);
  return true;
}

bool gemm_dx(const Dev& D, GemmState* g, cudaStream_t s) {
  if (!g || !D.dx) return false;
  const int G = D.cell == CAVS_CELL_TREE_LSTM ? 3 + D.N : 1;
  launch_rows<EPI_DX, kDxBN, 1>(g->A_dz, g->B_dx, D, G * D.h, 0, 0, D.d, s);
  return true;
}

}  // namespace cavs
