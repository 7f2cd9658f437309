// fw.cu — tiled blocked Floyd–Warshall on sm_100a.
//
// The cold-start comparator of the paper and the dense
// fallback of the removal algorithm ("If the Cost is larger than
// hyper-parameter delta, we just use the Floyd-Warshall algorithm").
//
// For each pivot block K of TB=128 nodes:
//   (1) fw_diag:  D_KK := FW closure of the 128x128 diagonal tile (one CTA,
//                 tile resident in shared memory, one barrier per pivot).
//   (2) panels:   D[K][J] := D_KK (x) D[K][J] and D[I][K] := D[I][K] (x) D_KK.
//                 One min-plus product with the closed tile — exact because a
//                 path between K and J decomposes at its last visit to K.
//   (3) rest:     D[I][J] := min(D[I][J], D[I][K] (x) D[K][J]), I, J != K.
// Steps (2) and (3) are the same register-tiled min-plus kernel: a 128x128
// output tile per CTA, 256 threads x (8x8) accumulators, k staged through
// shared memory in chunks of 32 (B tile by cp.async, A tile transposed
// through registers so every inner-loop operand is one LDS.128).  The int32
// relaxation min(d, a + b) is a single VIADDMNMX on sm_100a; no tensor cores
// (min-plus is not a (+,x) contraction).
#include "common.cuh"
#include "kernels.h"

namespace apsp {

constexpr int TB = 128;        // tile edge = pivot block
constexpr int KC = 32;         // k chunk staged in smem
constexpr int NTH = 256;       // threads per tile CTA
constexpr int AST = TB + 4;    // As row stride (elements), keeps LDS.128 aligned

// ---------------------------------------------------------------------------
// (1) closure of the diagonal tile
// ---------------------------------------------------------------------------
template <typename T, int SR>
__global__ void __launch_bounds__(1024) fw_diag_kernel(T* __restrict__ D, int64_t ld, int kb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T (*s)[TB] = reinterpret_cast<T (*)[TB]>(smem_raw);   // 64 KB tile
  const T I = Tr<T>::inf();
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    int i = e / TB, j = e % TB;
    s[i][j] = (i < kb && j < kb) ? D[(int64_t)i * ld + j] : I;
  }
  __syncthreads();
  // Row k and column k are unchanged by pivot k (D[k][k] = 0, w >= 0), so
  // the in-place update has no read/write race.
  for (int k = 0; k < kb; ++k) {
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
      int i = e / TB, j = e % TB;
      s[i][j] = Tr<T, SR>::relax(s[i][j], s[i][k], s[k][j]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    int i = e / TB, j = e % TB;
    if (i < kb && j < kb) D[(int64_t)i * ld + j] = s[i][j];
  }
}

// ---------------------------------------------------------------------------
// (2)/(3) C[I][J] = min(C[I][J], A[I][:] (x) B[:][J]) on 128x128 tiles
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_wait_all() { cp_async_wait<0>(); }   // common.cuh

struct TileArgs {
  void* C; int64_t ldc;          // output rows [0, m), cols [0, ncols)
  const void* A; int64_t lda;    // m x kdepth   (rows aligned with C)
  const void* B; int64_t ldb;    // kdepth x ncols
  int m, ncols, kdepth;
  int skip_ti, skip_tj;          // tile row / column excluded from this launch (-1: none)
};

template <typename T, int SR>
__global__ void __launch_bounds__(NTH, 1) fw_tile_kernel(TileArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);          // [2][KC][AST]   (k-major: As[k][i])
  T* Bs = As + 2 * KC * AST;                       // [2][KC][TB]    (Bs[k][j])

  const int tj = blockIdx.x, ti = blockIdx.y;
  if (ti == a.skip_ti || tj == a.skip_tj) return;
  T* C = reinterpret_cast<T*>(a.C);
  const T* A = reinterpret_cast<const T*>(a.A);
  const T* B = reinterpret_cast<const T*>(a.B);
  const T I = Tr<T>::inf();

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int i0 = ti * TB, j0 = tj * TB;
  const bool fullB = (j0 + TB <= a.ncols);
  const bool fullA = (i0 + TB <= a.m);
  const int nch = (a.kdepth + KC - 1) / KC;

  // --- staging helpers ---
  Vec4<T> areg[4];
  auto load_A = [&](int kc) {
    const int k0 = kc * KC;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + NTH * q;
      int r = idx >> 3, c4 = idx & 7;
      int kcol = k0 + c4 * 4;
      Vec4<T> v{I, I, I, I};
      if ((fullA || i0 + r < a.m) && kcol < a.kdepth) {
        v = ld4<T>(A + (int64_t)(i0 + r) * a.lda + kcol);
        v = mask_tail<T>(v, kcol, a.kdepth);
      }
      areg[q] = v;
    }
  };
  auto store_A = [&](int buf) {
    T* as = As + buf * KC * AST;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + NTH * q;
      int r = idx >> 3, c4 = idx & 7;
      as[(c4 * 4 + 0) * AST + r] = areg[q].x;
      as[(c4 * 4 + 1) * AST + r] = areg[q].y;
      as[(c4 * 4 + 2) * AST + r] = areg[q].z;
      as[(c4 * 4 + 3) * AST + r] = areg[q].w;
    }
  };
  auto load_B = [&](int kc, int buf) {
    const int k0 = kc * KC;
    T* bs = Bs + buf * KC * TB;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + NTH * q;
      int r = idx >> 5, c4 = idx & 31;
      int kr = k0 + r, col = j0 + c4 * 4;
      T* dst = bs + r * TB + c4 * 4;
      if (kr < a.kdepth && (fullB || col + 4 <= a.ncols)) {
        cp_async16(dst, B + (int64_t)kr * a.ldb + col);
      } else {
        Vec4<T> v{I, I, I, I};
        if (kr < a.kdepth && col < a.ncols) {
          v = ld4<T>(B + (int64_t)kr * a.ldb + col);
          v = mask_tail<T>(v, col, a.ncols);
        }
        st4<T>(dst, v);
      }
    }
    cp_async_commit();
  };

  // --- accumulators start from C ---
  T acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int row = i0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int col = j0 + (h == 0 ? tx * 4 : 64 + tx * 4);
      Vec4<T> v{I, I, I, I};
      if ((fullA || row < a.m) && (fullB || col < a.ncols)) v = ld4<T>(C + (int64_t)row * a.ldc + col);
      acc[r][h * 4 + 0] = v.x; acc[r][h * 4 + 1] = v.y;
      acc[r][h * 4 + 2] = v.z; acc[r][h * 4 + 3] = v.w;
    }
  }

  load_A(0);
  load_B(0, 0);
  store_A(0);
  cp_async_wait_all();
  __syncthreads();

  for (int kc = 0; kc < nch; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nch) {
      load_A(kc + 1);
      load_B(kc + 1, buf ^ 1);
    }
    const T* as = As + buf * KC * AST;
    const T* bs = Bs + buf * KC * TB;
    if constexpr (!(Tr<T>::kFloat && SR == 0)) {
      // int32: one VIADDMNMX per relaxation
#pragma unroll 8
      for (int kk = 0; kk < KC; ++kk) {
        Vec4<T> a0 = *reinterpret_cast<const Vec4<T>*>(as + kk * AST + ty * 4);
        Vec4<T> a1 = *reinterpret_cast<const Vec4<T>*>(as + kk * AST + 64 + ty * 4);
        Vec4<T> b0 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + tx * 4);
        Vec4<T> b1 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + 64 + tx * 4);
        T av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        T bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = Tr<T, SR>::relax(acc[r][c], av[r], bv[c]);
      }
    } else {
      // fp32: two pivots per step so each accumulator takes one 3-input
      // FMNMX3 per two FADDs (1.5 instructions per relaxation)
#pragma unroll 4
      for (int kk = 0; kk < KC; kk += 2) {
        Vec4<T> a0 = *reinterpret_cast<const Vec4<T>*>(as + kk * AST + ty * 4);
        Vec4<T> a1 = *reinterpret_cast<const Vec4<T>*>(as + kk * AST + 64 + ty * 4);
        Vec4<T> b0 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + tx * 4);
        Vec4<T> b1 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + 64 + tx * 4);
        Vec4<T> a2 = *reinterpret_cast<const Vec4<T>*>(as + (kk + 1) * AST + ty * 4);
        Vec4<T> a3 = *reinterpret_cast<const Vec4<T>*>(as + (kk + 1) * AST + 64 + ty * 4);
        Vec4<T> b2 = *reinterpret_cast<const Vec4<T>*>(bs + (kk + 1) * TB + tx * 4);
        Vec4<T> b3 = *reinterpret_cast<const Vec4<T>*>(bs + (kk + 1) * TB + 64 + tx * 4);
        T av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        T bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        T aw[8] = {a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
        T bw[8] = {b2.x, b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            acc[r][c] = fminf(acc[r][c], fminf(__fadd_rn(av[r], bv[c]), __fadd_rn(aw[r], bw[c])));
      }
    }
    if (kc + 1 < nch) store_A(buf ^ 1);
    cp_async_wait_all();
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int row = i0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4));
    if (!(fullA || row < a.m)) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int col = j0 + (h == 0 ? tx * 4 : 64 + tx * 4);
      if (!(fullB || col < a.ncols)) continue;
      Vec4<T> v{acc[r][h * 4 + 0], acc[r][h * 4 + 1], acc[r][h * 4 + 2], acc[r][h * 4 + 3]};
      st4<T>(C + (int64_t)row * a.ldc + col, v);
    }
  }
}

// ---------------------------------------------------------------------------
// Phase 3, fast path: A comes from PT, the pivot column panel stored
// TRANSPOSED (PT[k][i] = D[i][K0 + k], rows of ldpt elements, padded with INF
// to whole tiles), so both operand tiles arrive with 16-byte cp.async in the
// layout the inner loop reads (As[k][i], Bs[k][j]) — no register staging and
// no shared-memory transposes.  Out-of-range B rows/columns are zero-filled:
// the matching A entries are INF, so INF + 0 cannot lower any output.
// ---------------------------------------------------------------------------
struct Tile3Args {
  void* C; int64_t ldc;          // output rows [0, m), cols [0, ncols)
  const void* PT; int64_t ldpt;  // kdepth (padded to TB) x round_up(m, TB)
  const void* B; int64_t ldb;    // kdepth x ncols (row panel)
  int m, ncols, kdepth;
  int skip_ti, skip_tj;
};

template <typename T, int SR>
__global__ void __launch_bounds__(NTH, 2) fw_tile3_kernel(Tile3Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);          // [2][KC][TB]
  T* Bs = As + 2 * KC * TB;                        // [2][KC][TB]
  const int tj = blockIdx.x, ti = blockIdx.y;
  if (ti == a.skip_ti || tj == a.skip_tj) return;
  T* C = reinterpret_cast<T*>(a.C);
  const T* PT = reinterpret_cast<const T*>(a.PT);
  const T* B = reinterpret_cast<const T*>(a.B);
  const T I = Tr<T>::inf();
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int i0 = ti * TB, j0 = tj * TB;
  const bool fullB = (j0 + TB <= a.ncols);
  const bool fullA = (i0 + TB <= a.m);
  const int nch = (a.kdepth + KC - 1) / KC;

  auto load_chunk = [&](int kc, int buf) {
    const int k0 = kc * KC;
    T* as = As + buf * KC * TB;
    T* bs = Bs + buf * KC * TB;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + NTH * q;
      const int r = idx >> 5, c4 = idx & 31;
      cp_async16(as + r * TB + c4 * 4, PT + (int64_t)(k0 + r) * a.ldpt + i0 + c4 * 4);
      const int kr = k0 + r, col = j0 + c4 * 4;
      const T* src = B + (int64_t)kr * a.ldb + col;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(bs + r * TB + c4 * 4);
      const int bytes = (kr < a.kdepth && (fullB || col < a.ncols)) ? 16 : 0;
      if (bytes == 0) src = B;   // any valid address; zero-filled
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
    }
    cp_async_commit();
  };

  load_chunk(0, 0);
  T acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int row = i0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = j0 + (h == 0 ? tx * 4 : 64 + tx * 4);
      Vec4<T> v{I, I, I, I};
      if ((fullA || row < a.m) && (fullB || col < a.ncols)) v = ld4<T>(C + (int64_t)row * a.ldc + col);
      acc[r][h * 4 + 0] = v.x; acc[r][h * 4 + 1] = v.y;
      acc[r][h * 4 + 2] = v.z; acc[r][h * 4 + 3] = v.w;
    }
  }
  cp_async_wait_all();
  __syncthreads();

  for (int kc = 0; kc < nch; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nch) load_chunk(kc + 1, buf ^ 1);
    const T* as = As + buf * KC * TB;
    const T* bs = Bs + buf * KC * TB;
    if constexpr (!(Tr<T>::kFloat && SR == 0)) {
#pragma unroll 4
      for (int kk = 0; kk < KC; ++kk) {
        Vec4<T> a0 = *reinterpret_cast<const Vec4<T>*>(as + kk * TB + ty * 4);
        Vec4<T> a1 = *reinterpret_cast<const Vec4<T>*>(as + kk * TB + 64 + ty * 4);
        Vec4<T> b0 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + tx * 4);
        Vec4<T> b1 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + 64 + tx * 4);
        T av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        T bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = Tr<T, SR>::relax(acc[r][c], av[r], bv[c]);
      }
    } else {
#pragma unroll 2
      for (int kk = 0; kk < KC; kk += 2) {
        Vec4<T> a0 = *reinterpret_cast<const Vec4<T>*>(as + kk * TB + ty * 4);
        Vec4<T> a1 = *reinterpret_cast<const Vec4<T>*>(as + kk * TB + 64 + ty * 4);
        Vec4<T> b0 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + tx * 4);
        Vec4<T> b1 = *reinterpret_cast<const Vec4<T>*>(bs + kk * TB + 64 + tx * 4);
        Vec4<T> a2 = *reinterpret_cast<const Vec4<T>*>(as + (kk + 1) * TB + ty * 4);
        Vec4<T> a3 = *reinterpret_cast<const Vec4<T>*>(as + (kk + 1) * TB + 64 + ty * 4);
        Vec4<T> b2 = *reinterpret_cast<const Vec4<T>*>(bs + (kk + 1) * TB + tx * 4);
        Vec4<T> b3 = *reinterpret_cast<const Vec4<T>*>(bs + (kk + 1) * TB + 64 + tx * 4);
        T av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        T bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        T aw[8] = {a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
        T bw[8] = {b2.x, b2.y, b2.z, b2.w, b3.x, b3.y, b3.z, b3.w};
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            acc[r][c] = fminf(acc[r][c], fminf(__fadd_rn(av[r], bv[c]), __fadd_rn(aw[r], bw[c])));
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int row = i0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4));
    if (!(fullA || row < a.m)) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = j0 + (h == 0 ? tx * 4 : 64 + tx * 4);
      if (!(fullB || col < a.ncols)) continue;
      Vec4<T> v{acc[r][h * 4 + 0], acc[r][h * 4 + 1], acc[r][h * 4 + 2], acc[r][h * 4 + 3]};
      st4<T>(C + (int64_t)row * a.ldc + col, v);
    }
  }
}

// PT[k][i] = D[i][K0 + k] for k < kb, i < m; INF for k in [kb, TB) or i in [m, mpad)
template <typename T>
__global__ void fw_transpose_panel_kernel(const T* D, int64_t ld, int64_t m, int64_t K0, int kb,
                                          T* PT, int64_t ldpt, int64_t mpad) {
  __shared__ T tile[32][33];
  const int64_t i0 = blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r;
    const int k = k0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < m && k < kb) ? D[i * ld + K0 + k] : Tr<T>::inf();
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r;
    const int64_t i = i0 + threadIdx.x;
    if (i < mpad) PT[(int64_t)k * ldpt + i] = tile[threadIdx.x][r];
  }
}

constexpr size_t kTileSmem = sizeof(int32_t) * (2 * KC * AST + 2 * KC * TB);

template <typename T, int SR>
static cudaError_t launch_tile_sr(const TileArgs& a, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fw_tile_kernel<T, SR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTileSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (a.m <= 0 || a.ncols <= 0) return cudaSuccess;
  dim3 grid((a.ncols + TB - 1) / TB, (a.m + TB - 1) / TB);
  fw_tile_kernel<T, SR><<<grid, NTH, kTileSmem, st>>>(a);
  return cudaGetLastError();
}
template <typename T>
static cudaError_t launch_tile(const TileArgs& a, int sr, cudaStream_t st) {
  return sr ? launch_tile_sr<T, 1>(a, st) : launch_tile_sr<T, 0>(a, st);
}

// ---------------------------------------------------------------------------
// host-side drivers
// ---------------------------------------------------------------------------
template <typename T, int SR>
static cudaError_t fw_diag_sr(T* Dkk, int64_t ld, int kb, cudaStream_t st) {
  static bool configured = false;
  constexpr int smem = TB * TB * sizeof(T);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fw_diag_kernel<T, SR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  fw_diag_kernel<T, SR><<<1, 1024, smem, st>>>(Dkk, ld, kb);
  return cudaGetLastError();
}
template <typename T>
cudaError_t fw_diag(T* Dkk, int64_t ld, int kb, int sr, cudaStream_t st) {
  return sr ? fw_diag_sr<T, 1>(Dkk, ld, kb, st) : fw_diag_sr<T, 0>(Dkk, ld, kb, st);
}

// Row panel D[K][*] (all columns except the K tile) := D_KK (x) D[K][*].
// `rowK` points at D[K0][0]; ncols = n.
template <typename T>
cudaError_t fw_row_panel(T* rowK, int64_t ld, int64_t K0, int kb, int64_t ncols, int sr, cudaStream_t st) {
  TileArgs a;
  a.C = rowK; a.ldc = ld;
  a.A = rowK + K0; a.lda = ld;        // closed diagonal tile
  a.B = rowK; a.ldb = ld;             // the panel itself (each CTA reads only its own tile)
  a.m = kb; a.ncols = (int)ncols; a.kdepth = kb;
  a.skip_ti = -1; a.skip_tj = (int)(K0 / TB);
  return launch_tile<T>(a, sr, st);
}

// Column panel D[rows][K] := D[rows][K] (x) D_KK for m local rows.
// `D` = local rows base, `Dkk` = the closed diagonal tile (any ld).
// skip_ti = the local tile row holding the diagonal tile (-1 if not local).
template <typename T>
cudaError_t fw_col_panel(T* D, int64_t ld, int64_t m, int64_t K0, int kb, const T* Dkk,
                         int64_t lddk, int skip_ti, int sr, cudaStream_t st) {
  TileArgs a;
  a.C = D + K0; a.ldc = ld;
  a.A = D + K0; a.lda = ld;
  a.B = Dkk; a.ldb = lddk;
  a.m = (int)m; a.ncols = kb; a.kdepth = kb;
  a.skip_ti = skip_ti; a.skip_tj = -1;
  return launch_tile<T>(a, sr, st);
}

// Phase 3 on m local rows: D[i][j] = min(D[i][j], D[i][K] (x) P[K][j]) where
// P is the row panel (kb x ncols, leading dimension ldp).

template <typename T>
cudaError_t fw_rest_pt(T* D, int64_t ld, int64_t m, int64_t ncols, int64_t K0, int kb, const T* P,
                       int64_t ldp, int skip_ti, T* PT, int64_t ldpt, int sr, cudaStream_t st) {
  if (m <= 0 || ncols <= 0) return cudaSuccess;
  const int64_t mpad = (m + TB - 1) / TB * TB;
  if (mpad > ldpt) return cudaErrorInvalidValue;
  fw_transpose_panel_kernel<T><<<dim3((unsigned)(mpad / 32), TB / 32), dim3(32, 8), 0, st>>>(
      D, ld, m, K0, kb, PT, ldpt, mpad);
  static bool configured[2] = {false, false};
  constexpr size_t smem = sizeof(T) * 4 * KC * TB;
  if (!configured[sr ? 1 : 0]) {
    cudaError_t e = cudaFuncSetAttribute(sr ? fw_tile3_kernel<T, 1> : fw_tile3_kernel<T, 0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[sr ? 1 : 0] = true;
  }
  Tile3Args a;
  a.C = D; a.ldc = ld;
  a.PT = PT; a.ldpt = ldpt;
  a.B = P; a.ldb = ldp;
  a.m = (int)m; a.ncols = (int)ncols; a.kdepth = kb;
  a.skip_ti = skip_ti; a.skip_tj = (int)(K0 / TB);
  dim3 grid((unsigned)((ncols + TB - 1) / TB), (unsigned)(mpad / TB));
  if (sr)
    fw_tile3_kernel<T, 1><<<grid, NTH, smem, st>>>(a);
  else
    fw_tile3_kernel<T, 0><<<grid, NTH, smem, st>>>(a);
  return cudaGetLastError();
}

// ===========================================================================
// int16x2 blocked FW (int32 API, shortest path, one GPU).
//
// The int32 relaxation is one VIADDMNMX per pair; VIADDMNMX.S16x2 relaxes two
// int16 pairs per instruction (K13: 2x the int32 rate).  The FW runs on a
// packed copy P of D (two columns per word) with every value saturated at
// SAT = 0x3FFF: stored values stay <= SAT (each update is a min with the old
// value) and a sum of two is <= 32766, so nothing overflows.  Every entry whose
// true distance is < SAT comes out exact (an induction over the pivots: the
// shortest restricted path's sub-paths are shorter, hence exact; any candidate
// through a saturated value is >= SAT); every other entry comes out == SAT.
// Back-conversion writes the exact entries and raises a flag on any SAT, and
// the caller then re-runs the int32 FW on D (whose unconverted entries are
// still walk lengths, so the result is exact either way).
//
// Per pivot block K the same three phases as above, all on packed words:
//   (1) closure of the diagonal tile (one CTA, packed in shared memory);
//   (2) row panel D[K][*] := D_KK (x) D[K][*], column panel D[*][K] :=
//       D[*][K] (x) D_KK — fw_tile3_kernel<uint32_t> with A = a transposed,
//       half-replicated copy (PT[k][i] = D[i][k] in both halves);
//   (3) D[I][J] := min(D[I][J], D[I][K] (x) D[K][J]) — fw_tile3_kernel<uint32_t>
//       on 128-row x 256-column tiles (128 words).
// Recomputing the K tiles inside (2)/(3) is harmless: D_KK is closed.
// ===========================================================================
constexpr uint32_t kSat16 = 0x3FFFu;
__device__ __forceinline__ uint32_t half16(uint32_t w, int hi) { return hi ? (w >> 16) : (w & 0xFFFFu); }
__device__ __forceinline__ uint32_t rep16(uint32_t v) { return v | (v << 16); }

// P[i][w] = (sat(D[i][2w]), sat(D[i][2w+1])), columns >= n saturated
__global__ void k_d32_to_p16(const int32_t* __restrict__ D, int64_t ld, int64_t m, int64_t n,
                             uint32_t* __restrict__ P, int64_t ldw) {
  const int64_t tot = m * ldw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ldw, w = e - i * ldw, j = 2 * w;
    const uint32_t lo = j < n ? (uint32_t)min(D[i * ld + j], (int32_t)kSat16) : kSat16;
    const uint32_t hi = j + 1 < n ? (uint32_t)min(D[i * ld + j + 1], (int32_t)kSat16) : kSat16;
    P[e] = lo | (hi << 16);
  }
}

// D[i][j] := P value where it is < SAT; flag any other saturated entry.  Row and
// column `skip` (a tombstoned node: INF in D already, isolated in the graph)
// are neither written nor flagged.
__global__ void k_p16_to_d32(const uint32_t* __restrict__ P, int64_t ldw, int64_t m, int64_t n,
                             int64_t row0, int32_t* __restrict__ D, int64_t ld, int64_t skip,
                             unsigned* flag) {
  const int64_t tot = m * n;
  unsigned f = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    if (i + row0 == skip || j == skip) continue;
    const uint32_t v = half16(P[i * ldw + (j >> 1)], (int)(j & 1));
    if (v < kSat16) D[i * ld + j] = (int32_t)v;
    else f = 1;
  }
  if (__any_sync(0xffffffffu, f) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// closure of the kb x kb diagonal tile at P (word pointer of its top-left)
__global__ void __launch_bounds__(1024) k_p16_diag(uint32_t* __restrict__ P, int64_t ldw, int kb) {
  __shared__ uint32_t s[TB][TB / 2];
  for (int e = threadIdx.x; e < TB * TB / 2; e += blockDim.x) {
    const int i = e / (TB / 2), w = e % (TB / 2);
    uint32_t v = rep16(kSat16);
    if (i < kb) {
      const uint32_t x = P[(int64_t)i * ldw + w];
      const uint32_t lo = 2 * w < kb ? (x & 0xFFFFu) : kSat16;
      const uint32_t hi = 2 * w + 1 < kb ? (x >> 16) : kSat16;
      v = lo | (hi << 16);
    }
    s[i][w] = v;
  }
  __syncthreads();
  // row k and column k do not change at pivot k (D[k][k] = 0): in place
  for (int k = 0; k < kb; ++k) {
    for (int e = threadIdx.x; e < TB * TB / 2; e += blockDim.x) {
      const int i = e / (TB / 2), w = e % (TB / 2);
      s[i][w] = __viaddmin_s16x2(rep16(half16(s[i][k >> 1], k & 1)), s[k][w], s[i][w]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < TB * TB / 2; e += blockDim.x) {
    const int i = e / (TB / 2), w = e % (TB / 2);
    if (i < kb && 2 * w < kb) {
      uint32_t v = s[i][w];
      if (2 * w + 1 >= kb) v = (v & 0xFFFFu) | (P[(int64_t)i * ldw + w] & 0xFFFF0000u);   // keep the neighbour column
      P[(int64_t)i * ldw + w] = v;
    }
  }
}

// PT[k][i] = rep(D[i][K0 + k]) for k < kb, i < m; rep(SAT) elsewhere (i < mpad, k < TB)
__global__ void k_p16_transpose_rep(const uint32_t* __restrict__ P, int64_t ldw, int64_t m, int64_t K0,
                                    int kb, uint32_t* __restrict__ PT, int64_t ldpt, int64_t mpad) {
  __shared__ uint32_t tile[32][33];
  const int64_t i0 = blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r;
    const int k = k0 + threadIdx.x;
    uint32_t v = kSat16;
    if (i < m && k < kb) {
      const int64_t c = K0 + k;
      v = half16(P[i * ldw + (c >> 1)], (int)(c & 1));
    }
    tile[r][threadIdx.x] = rep16(v);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r;
    const int64_t i = i0 + threadIdx.x;
    if (i < mpad) PT[(int64_t)k * ldpt + i] = tile[threadIdx.x][r];
  }
}

static cudaError_t tile3_p16(uint32_t* C, int64_t ldc, const uint32_t* PT, int64_t ldpt, const uint32_t* B,
                             int64_t ldb, int64_t m, int64_t ncols, int kdepth, int skip_ti, cudaStream_t st) {
  static bool configured = false;
  constexpr size_t smem = sizeof(uint32_t) * 4 * KC * TB;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fw_tile3_kernel<uint32_t, 0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (m <= 0 || ncols <= 0) return cudaSuccess;
  Tile3Args a;
  a.C = C; a.ldc = ldc;
  a.PT = PT; a.ldpt = ldpt;
  a.B = B; a.ldb = ldb;
  a.m = (int)m; a.ncols = (int)ncols; a.kdepth = kdepth;
  a.skip_ti = skip_ti; a.skip_tj = -1;
  const int64_t mpad = (m + TB - 1) / TB * TB;
  dim3 grid((unsigned)((ncols + TB - 1) / TB), (unsigned)(mpad / TB));
  fw_tile3_kernel<uint32_t, 0><<<grid, NTH, smem, st>>>(a);
  return cudaGetLastError();
}

// ---- launchers (the per-pivot host loop is fw16_impl in apsp_warm.cu, which
// also broadcasts the packed row panel when D is row-sharded) ----
cudaError_t p16_from_d32(const int32_t* D, int64_t ld, int64_t m, int64_t n, uint32_t* P, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_d32_to_p16<<<num_sms() * 8, 256, 0, st>>>(D, ld, m, n, P, ld / 2);
  return cudaGetLastError();
}
cudaError_t p16_to_d32(const uint32_t* P, int64_t ld, int64_t m, int64_t n, int64_t row0, int64_t skip,
                       int32_t* D, unsigned* flag, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_p16_to_d32<<<num_sms() * 8, 256, 0, st>>>(P, ld / 2, m, n, row0, D, ld, skip, flag);
  return cudaGetLastError();
}
cudaError_t p16_diag(uint32_t* Pkk, int64_t ld, int kb, cudaStream_t st) {
  k_p16_diag<<<1, 1024, 0, st>>>(Pkk, ld / 2, kb);
  return cudaGetLastError();
}
cudaError_t p16_transpose_rep(const uint32_t* P, int64_t ld, int64_t m, int64_t K0, int kb, uint32_t* PT,
                              int64_t ldpt, cudaStream_t st) {
  const int64_t mpad = (m + TB - 1) / TB * TB;
  if (mpad == 0) return cudaSuccess;
  if (mpad > ldpt) return cudaErrorInvalidValue;
  k_p16_transpose_rep<<<dim3((unsigned)(mpad / 32), TB / 32), dim3(32, 8), 0, st>>>(P, ld / 2, m, K0, kb, PT,
                                                                                    ldpt, mpad);
  return cudaGetLastError();
}
cudaError_t p16_tile3(uint32_t* C, int64_t ld, const uint32_t* PT, int64_t ldpt, const uint32_t* B, int64_t m,
                      int64_t n, int kdepth, int skip_ti, cudaStream_t st) {
  // C and B rows are packed rows of D (ld/2 words); n = columns of D covered
  return tile3_p16(C, ld / 2, PT, ldpt, B, ld / 2, m, (n + 1) / 2, kdepth, skip_ti, st);
}

#define INST(T)                                                                                  \
  template cudaError_t fw_diag<T>(T*, int64_t, int, int, cudaStream_t);                          \
  template cudaError_t fw_row_panel<T>(T*, int64_t, int64_t, int, int64_t, int, cudaStream_t);   \
  template cudaError_t fw_col_panel<T>(T*, int64_t, int64_t, int64_t, int, const T*, int64_t,    \
                                       int, int, cudaStream_t);                                  \
  template cudaError_t fw_rest_pt<T>(T*, int64_t, int64_t, int64_t, int64_t, int, const T*,       \
                                     int64_t, int, T*, int64_t, int, cudaStream_t);
INST(int32_t)
INST(float)
#undef INST

}  // namespace apsp
