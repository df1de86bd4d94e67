// S3 at n = 128 — prime-factor (Good–Thomas) DST-I pass on the fp64 tensor pipe (DMMA).
//
// X_k = Σ_{j=1}^{128} x_j sin(π j k / 129)  (the DST-I of the fast Poisson solver)
// is -½ Im of the length-258 DFT of the odd extension x̃ (x̃_0 = x̃_129 = 0, x̃_{258-j} = -x_j).
// 258 = 2·3·43 with coprime factors, so with the input map j = CRT(j1, j2, j3) (j ≡ j1 mod 2,
// j ≡ j2 mod 3, j ≡ j3 mod 43) and the output map k = (129 k1 + 86 k2 + 6 k3) mod 258 the DFT
// becomes a 2 x 3 x 43 three-dimensional DFT with no twiddle factors:
//   z[j1][j2][j3] = x̃[CRT(j1,j2,j3)],   odd symmetry  z[j1][-j2][-j3] = -z[j1][j2][j3].
// Length-43 stage, per j1 (w(j3) = z[j1][1][j3]):
//   σ(k3) = Σ_{j3=1}^{21} z[j1][0][j3] sin(2π j3 k3/43)                       (odd in k3)
//   A(k3) = w(0) + Σ_{j3=1}^{21} (w(j3) + w(43-j3)) cos(2π j3 k3/43)           (even)
//   B(k3) = Σ_{j3=1}^{21} (w(j3) - w(43-j3)) sin(2π j3 k3/43)                  (odd)
// 3- and 2-point stages (closed form, all purely imaginary):
//   τ(k2=0)/2 = σ + B,   τ(1)/2 = (σ - B/2) + (√3/2) A,   τ(2)/2 = (σ - B/2) - (√3/2) A
//   X_k = τ_{j1=0}/2 + (-1)^{k1} τ_{j1=1}/2.
// Work per line: 4 sine (21x21) and 2 cosine (22x22) contractions padded to 24x24 for DMMA.m8n8k4:
// 3456 MACs per 128 outputs (27 MAC/point) instead of 8192 for the folded dense matrix.
//
// Kernel: persistent CTAs over tiles of 32 columns x all 128 rows of the transform axis (PASS 0:
// x, stride n^2, columns = flat (y,z); PASS 1: y, stride n, columns = flat (x,z)).  Tiles stream in
// with cp.async into a double buffer whose rows are the PERMUTED slots of the CRT map (so every
// B fragment reads 4 consecutive slots: bank-conflict free with the ≡4 (mod 16) row pitch); the
// odd-extension signs are applied to B fragments with a sign-bit XOR.  12 warps per CTA: warp =
// (8-column n-tile, 8-row m-tile of k3); each runs the 6 products as 6 independent DMMA chains
// (~80 registers, so 2 CTAs = 24 warps per SM hide the LDS -> DMMA latency).  The length-43
// results are staged in the consumed tile and a warp-uniform butterfly (lane = column, k3 and
// every output index compile-time) writes coalesced 256-byte rows straight to global memory.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <utility>

#include <cooperative_groups.h>

#include "dpm_internal.h"

namespace {

constexpr int N = 128, NN = N * N;
constexpr int TC = 32;              // columns per tile
constexpr int NTILE_N = TC / 8;     // 8-column n-tiles per tile
constexpr int NWARP = 3 * NTILE_N;  // warp = (n-tile, m-tile)
constexpr int NTHR = NWARP * 32;
constexpr int LD = TC + 4;          // row pitch (doubles), ≡ 4 mod 16
// slot layout (130 rows): W0 | U0 | W1 | U1 | 2 zero rows.  Entry e (0..23) of the U blocks is slot
// UB + e with data at e = 1..21; the neighbours read at e = 0, 22, 23 are finite data or zero rows
// and meet zero columns of S.  W blocks hold w(0..42) at WB + j3.
constexpr int W0B = 0, U0B = 42, W1B = 64, U1B = 106, NSLOT = 130;
constexpr int TILE = NSLOT * LD;    // doubles per buffer
constexpr int ATAB = 2 * 3 * 6 * 32;  // A-fragment table entries (S and C', 3 m-tiles, 6 k-steps, 32 lanes)
// staging rows (after the MMAs, inside the consumed buffer): σ0, σ1, B0, B1 at k3 = 1..21 and
// A0, A1 at k3 = 0..21 -> 128 rows, so the two zero rows (128, 129) are never overwritten.
constexpr int RS0 = 0, RS1 = 21, RB0 = 42, RB1 = 63, RA0 = 84, RA1 = 106;

__constant__ uint8_t c_slot[N];     // slot of transform-axis row r (0-based; x_{r+1})
__constant__ uint32_t c_usign[2];   // bit e: U block j1, entry e is -x (odd extension)
__constant__ uint64_t c_wsign[2];   // bit j3: W block j1, entry j3 is -x

struct Tables {
  uint8_t slot[N];
  uint32_t usign[2];
  uint64_t wsign[2];
};

// CRT of (j mod 2, j mod 3, j mod 43) -> j in [0, 258)
int crt258(int j1, int j2, int j3) {
  for (int j = 0; j < 258; ++j)
    if (j % 2 == j1 && j % 3 == j2 && j % 43 == j3) return j;
  return -1;
}

Tables make_tables() {
  Tables t{};
  for (int r = 0; r < N; ++r) t.slot[r] = 255;
  auto place = [&](int slot, int j) {   // x̃_j -> slot; returns true if the entry is -x
    const int x = j < 129 ? j : 258 - j;
    t.slot[x - 1] = (uint8_t)slot;
    return j > 129;
  };
  for (int j1 = 0; j1 < 2; ++j1) {
    const int ub = j1 ? U1B : U0B, wb = j1 ? W1B : W0B;
    for (int e = 1; e <= 21; ++e)
      if (place(ub + e, crt258(j1, 0, e))) t.usign[j1] |= 1u << e;
    for (int j3 = 0; j3 < 43; ++j3)
      if (place(wb + j3, crt258(j1, 1, j3))) t.wsign[j1] |= 1ull << j3;
  }
  return t;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double flip(double v, uint32_t signbit) {   // signbit: 0 or 0x80000000
  return __hiloint2double(__double2hiint(v) ^ (int)signbit, __double2loint(v));
}

__device__ __forceinline__ void cp_async16(unsigned smem_addr, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// global offset of (transform-axis row r, column cg) inside one field
template <int PASS>
__device__ __forceinline__ size_t goff(int r, int cg) {
  if (PASS == 0) return (size_t)r * NN + cg;
  return (size_t)(cg >> 7) * NN + (size_t)r * N + (cg & (N - 1));
}

// A fragments of the two 24x24 matrices (exact argument reduction mod 43):
//   S[k3][e]  = sin(2π e k3/43)          k3, e in 1..21   (zero elsewhere)
//   C'[k3][e] = (√3/2) cos(2π e k3/43)   k3, e in 0..21
// tab[((mat*3 + mt)*6 + ks)*32 + lane] = entry (row 8mt + lane/4, column 4ks + lane%4).
__global__ void pfa_atab_kernel(double* tab) {
  const int mat = blockIdx.x / 18, mt = (blockIdx.x / 6) % 3, ks = blockIdx.x % 6, lane = threadIdx.x;
  const int k3 = 8 * mt + (lane >> 2), e = 4 * ks + (lane & 3);
  const double arg = 2.0 * (double)((e * k3) % 43) / 43.0;
  double v;
  if (mat == 0) v = (k3 <= 21 && e >= 1 && e <= 21) ? sinpi(arg) : 0.0;
  else v = (k3 <= 21 && e <= 21) ? 0.86602540378443864676 * cospi(arg) : 0.0;
  tab[blockIdx.x * 32 + lane] = v;
}

template <int PASS>
__device__ __forceinline__ void load_tile(double* buf, const uint8_t* slot, const double* src, int col0) {
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(buf);
  constexpr int PER_ROW = TC / 2;                  // 16-byte requests per row
  const int c = 2 * (threadIdx.x % PER_ROW);
  for (int r = threadIdx.x / PER_ROW; r < N; r += NTHR / PER_ROW)
    cp_async16(sbase + 8u * (unsigned)(slot[r] * LD + c), src + goff<PASS>(r, col0 + c));
}

// Butterfly of one k3 row for one column (lane): the six staged length-43 results -> the (up to)
// 12 outputs X_k whose CRT class has this k3 (or 43 - k3); k, validity and signs are constants.
template <int PASS, int K3>
__device__ __forceinline__ void bfly(const double* R, double* dcol) {
  constexpr size_t STRIDE = PASS == 0 ? (size_t)NN : (size_t)N;
  double s0 = 0.0, s1 = 0.0, b0 = 0.0, b1 = 0.0;   // σ(0) = B(0) = 0
  if (K3 > 0) {
    s0 = R[(RS0 + K3 - 1) * LD];
    s1 = R[(RS1 + K3 - 1) * LD];
    b0 = R[(RB0 + K3 - 1) * LD];
    b1 = R[(RB1 + K3 - 1) * LD];
  }
  const double a0 = R[(RA0 + K3) * LD], a1 = R[(RA1 + K3) * LD];
  const double P0 = s0 + b0, P1 = s1 + b1, Q0 = fma(-0.5, b0, s0), Q1 = fma(-0.5, b1, s1);
  const double V[2][3] = {{P0 + P1, (Q0 + Q1) + (a0 + a1), (Q0 + Q1) - (a0 + a1)},
                          {P0 - P1, (Q0 - Q1) + (a0 - a1), (Q0 - Q1) - (a0 - a1)}};
#pragma unroll
  for (int mir = 0; mir < 2; ++mir) {
    if (mir && K3 == 0) break;
    const int k3f = mir ? 43 - K3 : K3;
#pragma unroll
    for (int k1 = 0; k1 < 2; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2) {
        const int k = (129 * k1 + 86 * k2 + 6 * k3f) % 258;
        if (k < 1 || k > 128) continue;
        // mirror k3f = 43 - k3 flips σ and B (P, Q) but not A:  -Q ± A = -(Q ∓ A)
        const double v = !mir ? V[k1][k2] : (k2 == 0 ? -V[k1][0] : (k2 == 1 ? -V[k1][2] : -V[k1][1]));
        __stcg(dcol + (size_t)(k - 1) * STRIDE, v);
      }
  }
}

template <int PASS, int... K3>
__device__ __forceinline__ void bfly_list(const double* R, double* dcol, std::integer_sequence<int, K3...>) {
  (bfly<PASS, K3>(R, dcol), ...);
}

template <int PASS>
__global__ void __launch_bounds__(NTHR, 2)
dst128_pass_kernel(const double* __restrict__ in, double* __restrict__ out, int nfields,
                   const double* __restrict__ atab) {
  extern __shared__ __align__(16) double smem[];
  __shared__ uint8_t slot[N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kk = lane & 3, rq = lane >> 2;
  const int nt = warp % NTILE_N, mt = warp / NTILE_N;

  for (int r = threadIdx.x; r < N; r += NTHR) slot[r] = c_slot[r];
  for (int i = threadIdx.x; i < 2 * 2 * LD; i += NTHR)       // zero rows 128, 129 of both buffers
    smem[(i / (2 * LD)) * TILE + (128 + (i / LD) % 2) * LD + i % LD] = 0.0;
  double aS[6], aC[6];
#pragma unroll
  for (int ks = 0; ks < 6; ++ks) {
    aS[ks] = __ldg(atab + ((0 * 3 + mt) * 6 + ks) * 32 + lane);
    aC[ks] = __ldg(atab + ((1 * 3 + mt) * 6 + ks) * 32 + lane);
  }
  // per-ks sign bits of this thread's B-fragment entries e = 4ks + kk
  uint32_t su0 = 0, su1 = 0, sw0a = 0, sw0b = 0, sw1a = 0, sw1b = 0;
#pragma unroll
  for (int ks = 0; ks < 6; ++ks) {
    const int e = 4 * ks + kk;
    su0 |= ((c_usign[0] >> e) & 1u) << ks;
    su1 |= ((c_usign[1] >> e) & 1u) << ks;
    sw0a |= (uint32_t)((c_wsign[0] >> e) & 1u) << ks;
    sw1a |= (uint32_t)((c_wsign[1] >> e) & 1u) << ks;
    if (e >= 1) {
      sw0b |= (uint32_t)((c_wsign[0] >> (43 - e)) & 1u) << ks;
      sw1b |= (uint32_t)((c_wsign[1] >> (43 - e)) & 1u) << ks;
    }
  }
  const double keep0 = kk == 0 ? 0.0 : 1.0;   // Wp(0) = w(0): drop the w(43) partner at e = 0
  __syncthreads();

  constexpr int TPF = NN / TC;   // tiles per field
  const long ntiles = (long)nfields * TPF;
  const size_t field = (size_t)NN * N;
  long tile = blockIdx.x;
  if (tile < ntiles) {
    const int f = (int)(tile / TPF);
    load_tile<PASS>(smem, slot, in + (size_t)f * field, (int)(tile - (long)f * TPF) * TC);
  }
  cp_async_commit();
  const int bcol = nt * 8 + rq;           // B-fragment column within the tile
  for (int cur = 0; tile < ntiles; tile += gridDim.x, cur ^= 1) {
    const long nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      const int f = (int)(nxt / TPF);
      load_tile<PASS>(smem + (cur ^ 1) * TILE, slot, in + (size_t)f * field, (int)(nxt - (long)f * TPF) * TC);
    }
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    double* T = smem + cur * TILE;

    double sg0[2] = {0, 0}, sg1[2] = {0, 0}, bb0[2] = {0, 0}, bb1[2] = {0, 0}, aa0[2] = {0, 0}, aa1[2] = {0, 0};
#pragma unroll
    for (int ks = 0; ks < 6; ++ks) {
      const int e = 4 * ks + kk;
      const double u0 = flip(T[(U0B + e) * LD + bcol], ((su0 >> ks) & 1u) << 31);
      const double u1 = flip(T[(U1B + e) * LD + bcol], ((su1 >> ks) & 1u) << 31);
      const double w0a = flip(T[(W0B + e) * LD + bcol], ((sw0a >> ks) & 1u) << 31);
      double w0b = flip(T[(W0B + 43 - e) * LD + bcol], ((sw0b >> ks) & 1u) << 31);
      const double w1a = flip(T[(W1B + e) * LD + bcol], ((sw1a >> ks) & 1u) << 31);
      double w1b = flip(T[(W1B + 43 - e) * LD + bcol], ((sw1b >> ks) & 1u) << 31);
      if (ks == 0) {
        w0b *= keep0;
        w1b *= keep0;
      }
      dmma884(sg0, aS[ks], u0);
      dmma884(sg1, aS[ks], u1);
      dmma884(bb0, aS[ks], w0a - w0b);
      dmma884(bb1, aS[ks], w1a - w1b);
      dmma884(aa0, aC[ks], w0a + w0b);
      dmma884(aa1, aC[ks], w1a + w1b);
    }
    // Stage the length-43 results in this warp's own (column, row) block of the consumed tile, so
    // that the butterfly below runs with k3 uniform across each warp (lanes = columns).
    __syncthreads();   // every warp has read its B fragments from T
    {
      const int k3 = 8 * mt + rq;
      const int c = nt * 8 + 2 * kk;
      if (k3 >= 1 && k3 <= 21) {
        *reinterpret_cast<double2*>(T + (RS0 + k3 - 1) * LD + c) = make_double2(sg0[0], sg0[1]);
        *reinterpret_cast<double2*>(T + (RS1 + k3 - 1) * LD + c) = make_double2(sg1[0], sg1[1]);
        *reinterpret_cast<double2*>(T + (RB0 + k3 - 1) * LD + c) = make_double2(bb0[0], bb0[1]);
        *reinterpret_cast<double2*>(T + (RB1 + k3 - 1) * LD + c) = make_double2(bb1[0], bb1[1]);
      }
      if (k3 <= 21) {
        *reinterpret_cast<double2*>(T + (RA0 + k3) * LD + c) = make_double2(aa0[0], aa0[1]);
        *reinterpret_cast<double2*>(T + (RA1 + k3) * LD + c) = make_double2(aa1[0], aa1[1]);
      }
    }
    __syncthreads();
    // 2x3 butterfly + output map: lane = column, warp w handles k3 = w, w + 12 with every output
    // index and sign a compile-time constant (no per-element index arithmetic).
    const int f = (int)(tile / TPF);
    double* dcol = out + (size_t)f * field + goff<PASS>(0, (int)(tile - (long)f * TPF) * TC + lane);
    const double* R = T + lane;
    switch (warp) {
      case 0: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 0, 12>{}); break;
      case 1: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 1, 13>{}); break;
      case 2: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 2, 14>{}); break;
      case 3: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 3, 15>{}); break;
      case 4: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 4, 16>{}); break;
      case 5: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 5, 17>{}); break;
      case 6: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 6, 18>{}); break;
      case 7: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 7, 19>{}); break;
      case 8: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 8, 20>{}); break;
      case 9: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 9, 21>{}); break;
      case 10: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 10>{}); break;
      default: bfly_list<PASS>(R, dcol, std::integer_sequence<int, 11>{}); break;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Thread-per-column DFMA variant (default).  Same Good–Thomas factorisation, but every thread owns
// one column: the length-43 stage runs as exact-size 21x21 / 22x22 dot products (2732 DFMA per
// column vs 3456 padded DMMA MACs, no fragment shuffling) whose matrix entries are warp-uniform
// constants (sin / (√3/2)cos of 2πm/43, m = e·k3 mod 43) and whose CRT rows and odd-extension
// signs are compile-time constants.  A warp reads 32 consecutive columns, so every load and store
// is one coalesced 256-byte row.  Per warp, shared memory holds the 64 prepared inputs of the
// current half (IN) and the j1 = 0 butterfly operands (ST); the contraction streams IN in blocks
// of 8 k3 rows (24 accumulator chains, ~80 registers).  No barriers.
__constant__ double c_s43[43];   // sin(2π m/43)
__constant__ double c_c43[43];   // (√3/2) cos(2π m/43)

__host__ __device__ constexpr int crt_c(int j1, int j2, int j3) {
  int j = 0;
  while (!(j % 2 == j1 && j % 3 == j2 && j % 43 == j3)) ++j;
  return j;
}
// x̃_j (j = CRT(...), j != 0, 129) = ±x_{row+1}
__host__ __device__ constexpr int crow(int j) { return (j < 129 ? j : 258 - j) - 1; }
__host__ __device__ constexpr bool cneg(int j) { return j > 129; }


// z[j1][j2][e] for this lane's half j1 (0 for lanes 0-15, 1 for lanes 16-31), read from the warp's
// RAW copy of the tile ([128 rows][16 columns], natural row order): both CRT rows and signs are
// compile-time constants; the lane picks one with an integer select and applies the sign as a
// sign-bit XOR (no divergence, nothing on the fp64 pipe).
template <int J2, int E>
__device__ __forceinline__ double ldz2(const double* raw, bool hi) {
  constexpr int ja = crt_c(0, J2, E), jb = crt_c(1, J2, E);
  const double v = raw[(hi ? crow(jb) : crow(ja)) * 16];
  constexpr int sa = cneg(ja) ? (int)0x80000000 : 0, sb = cneg(jb) ? (int)0x80000000 : 0;
  return __hiloint2double(__double2hiint(v) ^ (hi ? sb : sa), __double2loint(v));
}

// IN layout per warp (16 KB): (pin, qin) pairs for e = 1..21 at (e-1)*64 + 2*lane, then wp for
// e = 0..21 at IN_W + e*32 + lane.
constexpr int IN_W = 21 * 64, IN_SIZE = IN_W + 22 * 32, RAW_SIZE = 128 * 16;

// Prepare this lane's half: pin(e) = u(e) + wm(e), qin(e) = u(e) - wm(e)/2 (e = 1..21), wp(e) (0..21)
// with u(e) = z[j1][0][e], w(j3) = z[j1][1][j3], wm(e) = w(e) - w(43-e), wp(e) = w(e) + w(43-e).
template <int... E>
__device__ __forceinline__ void prep_half2(const double* raw, bool hi, double* in, int lane,
                                           std::integer_sequence<int, E...>) {
  in[IN_W + lane] = ldz2<1, 0>(raw, hi);
  auto one = [&](auto ec) {
    constexpr int e = decltype(ec)::value;
    const double u = ldz2<0, e>(raw, hi);
    const double wa = ldz2<1, e>(raw, hi), wb = ldz2<1, 43 - e>(raw, hi);
    const double wm = wa - wb;
    *reinterpret_cast<double2*>(in + (e - 1) * 64 + 2 * lane) = make_double2(u + wm, fma(-0.5, wm, u));
    in[IN_W + e * 32 + lane] = wa + wb;
  };
  (one(std::integral_constant<int, E + 1>{}), ...);
}

// cp.async of one 16-column x 128-row tile (16-byte requests) into the warp's RAW buffer
template <int PASS>
__device__ __forceinline__ void load_raw(double* raw, const double* fieldbase, int c0, int lane) {
  const unsigned sb = (unsigned)__cvta_generic_to_shared(raw);
  const int cc = 2 * (lane & 7);
#pragma unroll 8
  for (int r = lane >> 3; r < N; r += 4)
    cp_async16(sb + 8u * (unsigned)(r * 16 + cc), fieldbase + goff<PASS>(r, c0 + cc));
}

// Contract one block of KB k3 rows starting at K0:  P = S·pin, Q = S·qin, R = C'·wp.
// `in` points at this lane's IN slot (pairs at in + IN_PQ + e*64 (+lane*2 folded by the caller)).
template <int K0, int KB, typename Emit>
__device__ __forceinline__ void contract_block(const double* inpq, const double* inw, Emit&& emit) {
  double P[KB], Q[KB], R[KB];
#pragma unroll
  for (int q = 0; q < KB; ++q) P[q] = Q[q] = R[q] = 0.0;
#pragma unroll
  for (int e = 0; e <= 21; ++e) {
    const double w = inw[e * 32];
    double2 pq = make_double2(0.0, 0.0);
    if (e >= 1) pq = *reinterpret_cast<const double2*>(inpq + (e - 1) * 64);
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int k3 = K0 + q;
      // only 22 + 21 distinct magnitudes (sin(2π(43-m)/43) = -sin, cos even): the compiler keeps
      // them in (uniform) registers and applies the sign as a free operand negation
      const int m = (e * k3) % 43;
      const double cm = m <= 21 ? c_c43[m] : c_c43[43 - m];
      R[q] = fma(w, cm, R[q]);
      if (e >= 1 && k3 >= 1) {
        const double sm = m <= 21 ? c_s43[m] : -c_s43[43 - m];
        P[q] = fma(pq.x, sm, P[q]);
        Q[q] = fma(pq.y, sm, Q[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < KB; ++q) emit(std::integral_constant<int, K0>{}, q, P[q], Q[q], R[q]);
}

// lanes 0-15: half j1 = 0 of columns 0..15; lanes 16-31: half j1 = 1 of the same columns.  The final
// 2-point stage X_k = T0 ± T1 pairs lane l with l ^ 16 (one shuffle per operand): lane l writes the
// k1 = 0 outputs, lane l + 16 the k1 = 1 outputs.  14 warps per SM, 16 KB of IN per warp.
// MODE 0: dense in / dense out.  MODE 1 (sparse in; the fused BEP build, bep_fused.cu, forward x
// pass): the tile is gathered from the compact band values of the field, stored x-line-major: per
// x-line L (= a column of the x pass) a 32-byte entry tab[L] = {128-bit mask of the x positions
// holding band points, start of the line's values}.  The tile is zeroed and only the set rows are
// copied (cp.async, issued for the next tile under the contraction): no zero-filled box is read.
// (A γ-out variant of the inverse pass, writing only the γ outputs through the γ line table, was
// measured slower than the dense inverse pass + gather: the per-output slot arithmetic adds ~40%
// instructions to this instruction-bound kernel.)
struct LineEntry {
  uint32_t m[4];
  int32_t start;
};

__device__ __forceinline__ LineEntry load_line(const uint32_t* __restrict__ tab, int line) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(tab) + 2 * (size_t)line);
  const int32_t st = __ldg(reinterpret_cast<const int32_t*>(tab) + 8 * (size_t)line + 4);
  return LineEntry{{a.x, a.y, a.z, a.w}, st};
}

// zero the tile, then cp.async (8-byte) only the band values of the lane's line into their rows;
// the two lanes of a column take alternate set bits.  Issued for the next tile under the contraction.
template <int PASS>
__device__ __forceinline__ void load_raw_lines(double* raw, const uint32_t* __restrict__ tab,
                                               const double* __restrict__ vals, int c0, int lane) {
  const int cc = lane & 15, h = lane >> 4;
#pragma unroll
  for (int i = 0; i < 16; ++i)   // 128 x 16 doubles: 4 per lane per 16-byte store
    *reinterpret_cast<double4*>(raw + (i * 32 + lane) * 4) = make_double4(0.0, 0.0, 0.0, 0.0);
  __syncwarp();
  const LineEntry e = load_line(tab, c0 + cc);
  const unsigned sb = (unsigned)__cvta_generic_to_shared(raw);
  int slot = e.start;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t m = e.m[w];
    for (int k = 0; m; ++k) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      if ((k & 1) == h)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + 8u * (unsigned)((32 * w + b) * 16 + cc)),
                     "l"(vals + slot + k));
    }
    slot += __popc(e.m[w]);
  }
}

template <int PASS, int MINB, int MODE = 0>
__global__ void __launch_bounds__(224, MINB)
dst128f_kernel(const double* __restrict__ in, double* __restrict__ out, int nfields,
               const uint32_t* __restrict__ tab = nullptr, const double* vals = nullptr, int64_t ldv = 0) {
  extern __shared__ __align__(16) double wsm[];   // [warp][IN 16 KB | RAW 16 KB]
  const int lane = threadIdx.x & 31;
  const bool hi = lane >= 16;
  double* wbase = wsm + (threadIdx.x >> 5) * (IN_SIZE + RAW_SIZE);
  double* raw = wbase + IN_SIZE;
  const double* inpq = wbase + 2 * lane;
  const double* inw = wbase + IN_W + lane;
  constexpr size_t STRIDE = PASS == 0 ? (size_t)NN : (size_t)N;
  constexpr int TPF = NN / 16;
  const int ntiles = nfields * TPF;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
  const double sm1 = hi ? -1.0 : 1.0;
  const size_t field = (size_t)NN * N;
  if (gw < ntiles) {
    const int f = gw / TPF;
    if (MODE == 1)
      load_raw_lines<PASS>(raw, tab, vals + (size_t)f * ldv, (gw - f * TPF) * 16, lane);
    else
      load_raw<PASS>(raw, in + (size_t)f * field, (gw - f * TPF) * 16, lane);
  }
  cp_async_commit();
  for (int t = gw; t < ntiles; t += nw) {
    const int f = t / TPF, cg = (t - f * TPF) * 16 + (lane & 15);
    double* ocol = out + (size_t)f * field + goff<PASS>(0, cg);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
    prep_half2(raw + (lane & 15), hi, wbase, lane, std::make_integer_sequence<int, 21>{});
    __syncwarp();   // RAW consumed: prefetch the next tile under the contraction
    const int tn = t + nw;
    if (tn < ntiles) {
      const int fn = tn / TPF;
      if (MODE == 1)
        load_raw_lines<PASS>(raw, tab, vals + (size_t)fn * ldv, (tn - fn * TPF) * 16, lane);
      else
        load_raw<PASS>(raw, in + (size_t)fn * field, (tn - fn * TPF) * 16, lane);
    }
    cp_async_commit();
    auto bfly = [&](auto k0c, int q, double P, double Q, double R) {
      const int k3 = decltype(k0c)::value + q;
      // lane l (j1 = 0) forms T0 + T1 (k1 = 0), lane l + 16 (j1 = 1) forms T0 - T1 (k1 = 1):
      //   X = other ± mine  ->  fma(±1, mine, other)
      const double Ps = fma(sm1, P, __shfl_xor_sync(0xffffffffu, P, 16));
      const double Qs = fma(sm1, Q, __shfl_xor_sync(0xffffffffu, Q, 16));
      const double Rs = fma(sm1, R, __shfl_xor_sync(0xffffffffu, R, 16));
      // (for the hi lane Ps = T0 - T1 exactly as the k1 = 1 formula needs)
      const double V[3] = {Ps, Qs + Rs, Qs - Rs};
#pragma unroll
      for (int mir = 0; mir < 2; ++mir) {
        if (mir && k3 == 0) break;
        const int k3f = mir ? 43 - k3 : k3;
#pragma unroll
        for (int k2 = 0; k2 < 3; ++k2) {
          const int ka = (86 * k2 + 6 * k3f) % 258, kb = (129 + 86 * k2 + 6 * k3f) % 258;
          const bool va = ka >= 1 && ka <= 128, vb = kb >= 1 && kb <= 128;
          if (!va && !vb) continue;
          // mirror k3f = 43 - k3 flips σ and B (P, Q) but not A:  -Q ± R = -(Q ∓ R)
          const double v = !mir ? V[k2] : (k2 == 0 ? -V[0] : (k2 == 1 ? -V[2] : -V[1]));
          if (hi ? vb : va) __stcg(ocol + (size_t)((hi ? kb : ka) - 1) * STRIDE, v);
        }
      }
    };
    // __syncwarp between blocks: keeps ptxas from interleaving the blocks' accumulator sets
    __syncwarp();
    contract_block<0, 8>(inpq, inw, bfly);
    __syncwarp();
    contract_block<8, 8>(inpq, inw, bfly);
    __syncwarp();
    contract_block<16, 6>(inpq, inw, bfly);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// Fused plane pass: after the x transform every x-mode plane a ([y][z], 128 x 128,
// contiguous) is independent.  One 2-CTA cluster per plane; CTA r holds columns z in [64r, 64r+64)
// of the plane in shared memory (pitch 65: conflict-free for both the column-wise transforms and
// the row-wise recurrences) and runs, on chip:
//   (1) y forward DST-I of its 64 columns (thread-per-column DFMA, same factorisation as above,
//       inputs held in registers so the outputs overwrite the column in place),
//   (2) the exact z tridiagonal solve of every y-mode row b, split at z = 64 between the two CTAs:
//       each CTA solves its half with a zero interface value, the halves exchange one boundary value
//       per row through distributed shared memory, solve the 2x2 interface system and add the
//       closed-form homogeneous responses g_L[k] = μ^{64-k}(1-μ^{2(k+1)})/(1-μ^{130}), g_R[k] = g_L[63-k],
//   (3) y inverse DST-I,
// replacing three streaming passes over the field (y, z, y) by one.
#ifndef PLANE_KB
#define PLANE_KB 6
#endif
constexpr int PHC = 64;          // columns per CTA
constexpr int PPITCH = 65;       // row pitch (doubles)
constexpr int PTHR = 128;        // 4 warps x 16 columns x 2 halves

template <int J2, int E>
__device__ __forceinline__ double ldzp(const double* colp, bool hi) {
  constexpr int ja = crt_c(0, J2, E), jb = crt_c(1, J2, E);
  const double v = colp[(hi ? crow(jb) : crow(ja)) * PPITCH];
  constexpr int sa = cneg(ja) ? (int)0x80000000 : 0, sb = cneg(jb) ? (int)0x80000000 : 0;
  return __hiloint2double(__double2hiint(v) ^ (hi ? sb : sa), __double2loint(v));
}

template <int... E>
__device__ __forceinline__ void prep_regs(const double* colp, bool hi, double (&pin)[22], double (&qin)[22],
                                          double (&wp)[22], std::integer_sequence<int, E...>) {
  wp[0] = ldzp<1, 0>(colp, hi);
  pin[0] = qin[0] = 0.0;
  auto one = [&](auto ec) {
    constexpr int e = decltype(ec)::value;
    const double u = ldzp<0, e>(colp, hi);
    const double wa = ldzp<1, e>(colp, hi), wb = ldzp<1, 43 - e>(colp, hi);
    const double wm = wa - wb;
    pin[e] = u + wm;
    qin[e] = fma(-0.5, wm, u);
    wp[e] = wa + wb;
  };
  (one(std::integral_constant<int, E + 1>{}), ...);
}

template <int K0, int KB, typename Emit>
__device__ __forceinline__ void contract_regs(const double (&pin)[22], const double (&qin)[22],
                                              const double (&wp)[22], Emit&& emit) {
  double P[KB], Q[KB], R[KB];
#pragma unroll
  for (int q = 0; q < KB; ++q) P[q] = Q[q] = R[q] = 0.0;
#pragma unroll
  for (int e = 0; e <= 21; ++e)
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int k3 = K0 + q;
      const int m = (e * k3) % 43;
      const double cm = m <= 21 ? c_c43[m] : c_c43[43 - m];
      R[q] = fma(wp[e], cm, R[q]);
      if (e >= 1 && k3 >= 1) {
        const double sm = m <= 21 ? c_s43[m] : -c_s43[43 - m];
        P[q] = fma(pin[e], sm, P[q]);
        Q[q] = fma(qin[e], sm, Q[q]);
      }
    }
#pragma unroll
  for (int q = 0; q < KB; ++q) emit(std::integral_constant<int, K0>{}, q, P[q], Q[q], R[q]);
}

// In-place DST-I along the rows (y) of this CTA's 64 columns (KEPT = false: thread = (column, CRT
// half)), or of the 32 kept columns 0..31 only (KEPT = true, FACR(1) below: thread = (column, CRT
// half, k3 group); the two k3 groups split the contraction 11/11).
// (KEPT: one out-of-line copy shared by the forward and inverse transforms keeps the FACR kernel's
// code within the instruction cache.)
#ifndef PLANE_YDST_INLINE
#define PLANE_YDST_INLINE 0
#endif
template <bool KEPT>
__device__ __noinline__ void plane_ydst_call(double* P);
template <bool KEPT>
__device__ __forceinline__ void plane_ydst(double* P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool hi = lane >= 16;
  const int col = KEPT ? (warp & 1) * 16 + (lane & 15) : warp * 16 + (lane & 15);
  double* colp = P + col;
  double pin[22], qin[22], wp[22];
  prep_regs(colp, hi, pin, qin, wp, std::make_integer_sequence<int, 21>{});
  if (KEPT)
    __syncthreads();   // all four threads of every column have read their inputs
  else
    __syncwarp();      // both halves of every column have read their inputs: outputs may overwrite it
  const double sm1 = hi ? -1.0 : 1.0;
  auto bfly = [&](auto k0c, int q, double Pv, double Qv, double Rv) {
    const int k3 = decltype(k0c)::value + q;
    const double Ps = fma(sm1, Pv, __shfl_xor_sync(0xffffffffu, Pv, 16));
    const double Qs = fma(sm1, Qv, __shfl_xor_sync(0xffffffffu, Qv, 16));
    const double Rs = fma(sm1, Rv, __shfl_xor_sync(0xffffffffu, Rv, 16));
    const double V[3] = {Ps, Qs + Rs, Qs - Rs};
#pragma unroll
    for (int mir = 0; mir < 2; ++mir) {
      if (mir && k3 == 0) break;
      const int k3f = mir ? 43 - k3 : k3;
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2) {
        const int ka = (86 * k2 + 6 * k3f) % 258, kb = (129 + 86 * k2 + 6 * k3f) % 258;
        const bool va = ka >= 1 && ka <= 128, vb = kb >= 1 && kb <= 128;
        if (!va && !vb) continue;
        const double v = !mir ? V[k2] : (k2 == 0 ? -V[0] : (k2 == 1 ? -V[2] : -V[1]));
        if (hi ? vb : va) colp[((hi ? kb : ka) - 1) * PPITCH] = v;
      }
    }
  };
  if (KEPT) {
    if (warp >> 1) {
      contract_regs<11, 6>(pin, qin, wp, bfly);
      __syncwarp();
      contract_regs<17, 5>(pin, qin, wp, bfly);
    } else {
      contract_regs<0, 6>(pin, qin, wp, bfly);
      __syncwarp();
      contract_regs<6, 5>(pin, qin, wp, bfly);
    }
    return;
  }
#if PLANE_KB == 8
  contract_regs<0, 8>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<8, 8>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<16, 6>(pin, qin, wp, bfly);
  __syncwarp();
#elif PLANE_KB == 4
  contract_regs<0, 4>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<4, 4>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<8, 4>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<12, 4>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<16, 4>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<20, 2>(pin, qin, wp, bfly);
  __syncwarp();
#else
  contract_regs<0, 6>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<6, 6>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<12, 6>(pin, qin, wp, bfly);
  __syncwarp();
  contract_regs<18, 4>(pin, qin, wp, bfly);
  __syncwarp();
#endif
}

template <bool KEPT>
__device__ __noinline__ void plane_ydst_call(double* P) {
  plane_ydst<KEPT>(P);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHR, 2)
plane128_kernel(double* __restrict__ u, const double* __restrict__ lam_g, double inv_dt, double h2, double rscale) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double psm[];
  double* P = psm;                           // [128 rows][PPITCH]
  double* lam = psm + N * PPITCH;            // [128]
  double* xch = lam + N;                     // [128] boundary value received from the partner
  const int rank = (int)cluster.block_rank();
  const long plane = blockIdx.x >> 1;        // field * 128 + a
  const int a = (int)(plane & (N - 1));
  double* gp = u + (size_t)plane * NN + (size_t)rank * PHC;
  for (int i = threadIdx.x; i < N; i += PTHR) lam[i] = lam_g[i];
  // load the half plane: rows of 64 contiguous doubles, 8-byte cp.async (all in flight at once)
  {
    const unsigned sb = (unsigned)__cvta_generic_to_shared(P);
#pragma unroll 16
    for (int e = threadIdx.x; e < N * PHC; e += PTHR) {
      const int r = e >> 6, c = e & 63;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + 8u * (unsigned)(r * PPITCH + c)),
                   "l"(gp + (size_t)r * N + c));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  plane_ydst<false>(P);
  __syncthreads();
  // z tridiagonal per y-mode row b = threadIdx.x, on this CTA's half (local k = 0..63)
  {
    const int b = threadIdx.x;
    double* row = P + b * PPITCH;
    const double hs = h2 * ((inv_dt + lam[a]) + lam[b]);
    const double disc = sqrt(hs * (hs + 4.0));
    const double mu = 2.0 / ((2.0 + hs) + disc);
    constexpr int M = PHC;
    // A^{-1} r = μ z: forward y_k = r_k + μ y_{k-1}, backward z_k = y_k + μ z_{k+1}
    double y = 0.0;
    for (int k = 0; k < M; ++k) {
      y = fma(mu, y, rscale * row[k]);
      row[k] = y;
    }
    double z = 0.0;
    for (int k = M - 1; k >= 0; --k) {
      z = fma(mu, z, row[k]);
      row[k] = z;
    }
    // local Dirichlet solve x_k = μ z_k - c2 (μ^{k+1} - μ^{2M+1-k}),  c2 = μ^2 z_0 / (1 - μ^{2M+2});
    // only the interface entry is needed before the exchange (x_63 left, x_0 right)
    double muM = mu;                                       // μ^M, M = 64 = 2^6
#pragma unroll
    for (int q = 0; q < 6; ++q) muM *= muM;
    const double mu2M1 = muM * muM * mu;                   // μ^{2M+1}
    const double den = 1.0 - mu2M1 * mu;                   // 1 - μ^{2M+2}
    const double c2 = mu * mu * row[0] / den;
    const double mine = rank == 0 ? fma(mu, row[M - 1], -c2 * (muM - muM * mu * mu))   // k = 63
                                  : fma(mu, row[0], -c2 * (mu - mu2M1));                // k = 0
    // interface: left half (rank 0) owns z = 63 (local 63), right half (rank 1) owns z = 64 (local 0)
    double* peer = cluster.map_shared_rank(xch, rank ^ 1);
    peer[b] = mine;
    cluster.sync();
    const double other = xch[b];
    const double x63 = rank == 0 ? mine : other, y0 = rank == 0 ? other : mine;
    const double gam = mu * (1.0 - muM * muM) / den;       // g_L[63] = g_R[0]
    const double v63 = (x63 + y0 * gam) / (1.0 - gam * gam);
    const double v64 = y0 + v63 * gam;
    const double w = (rank == 0 ? v64 : v63) / den;
    // final: v_k = μ z_k - c2 (μ^{k+1} - μ^{2M+1-k}) + w (g1_k - g2_k) with the homogeneous response
    //   left  g_L[k] den = μ^{M-k} - μ^{M+k+2},   right g_R[k] den = μ^{k+1} - μ^{2M+1-k}
    // (the right response is the same power pair as the Sherman–Morrison term).  Every running
    // power whose term matters is walked in the direction in which it shrinks (pa, and the right
    // response, ascending; the left response descending), so an underflowed start (μ^M < 1e-308
    // at tiny dt) can only drop terms that are themselves below 1e-150 of the solution.
    const double imu = 1.0 / mu;
    const double A = rank == 0 ? -c2 : w - c2;             // coefficient of (μ^{k+1} - μ^{2M+1-k})
    double pa = mu, pb = mu2M1;                            // μ^{k+1}, μ^{2M+1-k}
    for (int k = 0; k < M; ++k) {
      row[k] = fma(mu, row[k], A * (pa - pb));
      pa *= mu;
      pb *= imu;
    }
    if (rank == 0) {
      double ga = mu, gb = mu2M1;                          // μ^{M-k}, μ^{M+k+2} at k = M-1
      for (int k = M - 1; k >= 0; --k) {
        row[k] = fma(w, ga - gb, row[k]);
        ga *= mu;
        gb *= imu;
      }
    }
  }
  __syncthreads();
  plane_ydst<false>(P);
  __syncthreads();
  for (int e = threadIdx.x; e < N * PHC; e += PTHR) {
    const int r = e >> 6, c = e & 63;
    __stcg(gp + (size_t)r * N + c, P[r * PPITCH + c]);
  }
  // (all DSMEM writes into this CTA completed before the cluster barrier above)
}

// ---------------------------------------------------------------------------------------------
// FACR(1) plane pass ("plane pass, FACR(1)"): the same per-plane problem
//   T_y v_z - v_{z-1} - v_{z+1} = g_z,   T_y = tridiag(-1, β, -1) along y,  β = 4 + h²(1/dt + λ_a),
// with one level of cyclic reduction along z before the transform.  Adding T_y·(row z) to rows z±1
// for odd z (0-based) eliminates the even z and leaves, for the 64 odd ("kept") z,
//   -v_{z-2} + (T_y² - 2) v_z - v_{z+2} = T_y g_z + g_{z-1} + g_{z+1}      (z = 127: T_y² - 1)
// which the y DST-I diagonalises with eigenvalues τ_b² - 2, τ_b = 2 + h²(1/dt + λ_a + λ_b).  The
// y transforms thus run on 32 columns per CTA instead of 64; the even z are recovered afterwards
// from  T_y v_z = g_z + v_{z-1} + v_{z+1}  (constant-coefficient tridiagonal solves along y).
// Phases per CTA (rank r holds z in [64r, 64r+64); smem columns 0..31 = kept z (odd), 32..63 =
// eliminated z (even), column 64 = the neighbour column):
//   (1) reduced right-hand side on the kept columns (rank 0 also loads z = 64 from global memory),
//   (2) y DST-I of the 32 kept columns (one out-of-line copy of the transform, 4 threads/column),
//   (3) reduced tridiagonal per y-mode row, in registers (32 unknowns per CTA, split exactly as in
//       plane128_kernel; the last row of rank 1 carries the extra +1 by Sherman–Morrison),
//   (4) inverse y DST-I of the kept columns; rank 0 pushes v(z = 63) into rank 1's column 64,
//   (5) eliminated columns: y tridiagonal solves in registers, 4 lanes per column over row
//       segments [0,33) [33,64) [64,97) [97,128), forward/backward carries by warp shuffles.
// Measured (profiles/r01/ncu_plane128_facr_full.txt): 0.77 ms per 64 fields vs 0.86 ms for
// plane128_kernel; 30% fewer instructions, DFMA count -40%.
// Running powers of μ are only walked in the direction in which they shrink when their term is
// not negligible (see plane128_kernel).
[[maybe_unused]] __device__ __forceinline__ double ipow128(double b, int e) {   // b^e, 0 <= e < 512
  double r = 1.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if ((e >> q) & 1) r *= b;
    b *= b;
  }
  return r;
}

// Cluster signalling without GPU-scope fences: the sender writes the partner's shared memory with
// st.async, which completes a transaction count on the partner's mbarrier; the receiver waits on
// its own mbarrier.  (barrier.cluster.arrive.release lowers to MEMBAR.ALL.GPU + ERRBAR: ~5% of the
// kernel's stall samples in the first version.)
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ unsigned mapa(unsigned local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(unsigned remote, double v, unsigned remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(remote),
               "l"(__double_as_longlong(v)), "r"(remote_bar)
               : "memory");
}

// Optional phase timing (build with -DFACR_PHASE_TIMING=1, read with dpm_debug_facr_phases; not in
// the default library): clock64 at the phase boundaries of the first FACR_TCTAS CTAs, thread 0.
#ifndef FACR_PHASE_TIMING
#define FACR_PHASE_TIMING 0
#endif
// Phase 5 with the four running powers of its correction merged into two and the powers of μ from shared
// squarings (0: the first form, four walks and five ipow128 calls)
// unroll depth of the final store loop (shared-memory loads in flight ahead of the global stores)
#ifndef PLANE_STORE_UNROLL
#define PLANE_STORE_UNROLL 4
#endif
#ifndef PLANE_STORE_CS
#define PLANE_STORE_CS 0   // 1: st.global.cs (evict-first) for the plane's output
#endif
#define PLANE_PRAGMA(x) _Pragma(#x)
#define PLANE_UNROLL(n) PLANE_PRAGMA(unroll n)
#ifndef PLANE_P5_MERGED
#define PLANE_P5_MERGED 1
#endif
constexpr int FACR_TCTAS = 4096, FACR_TPH = 9;
// Speed-of-light switches (timing experiments only, tools/plane_sol.sh; results are wrong when any is
// set): skip the half-plane load, phase 1, the two transforms, the phase-3 recurrences, phase 5 or
// the store.
#ifndef PLANE_SOL_NOLOAD
#define PLANE_SOL_NOLOAD 0
#endif
#ifndef PLANE_SOL_NOP1
#define PLANE_SOL_NOP1 0
#endif
#ifndef PLANE_SOL_NOXF
#define PLANE_SOL_NOXF 0
#endif
#ifndef PLANE_SOL_NOP3
#define PLANE_SOL_NOP3 0
#endif
#ifndef PLANE_SOL_NOP5
#define PLANE_SOL_NOP5 0
#endif
#ifndef PLANE_SOL_NOSTORE
#define PLANE_SOL_NOSTORE 0
#endif
#if FACR_PHASE_TIMING
__device__ unsigned long long g_facr_ph[FACR_TCTAS][FACR_TPH];
#define FACR_MARK(k)                                                              \
  do {                                                                            \
    if (threadIdx.x == 0 && blockIdx.x < FACR_TCTAS) g_facr_ph[blockIdx.x][k] = clock64(); \
  } while (0)
#else
#define FACR_MARK(k) \
  do {               \
  } while (0)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHR, 2)
plane128_facr_kernel(double* __restrict__ u, const double* __restrict__ lam_g, double inv_dt, double h2,
                     double gs) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double psm[];
  // P[row y][col]: kept z = 2i+1 (local) at col i (0..31), eliminated z = 2j at col 32 + j, col 64:
  // the neighbour column (phase 1: z = 64 for rank 0 / ghost z = 128 for rank 1; phase 5: v at
  // z = 63 for rank 1 / ghost z = -1 for rank 0).  Consecutive lanes touch consecutive columns in
  // every phase (bank-conflict free with the odd pitch).
  double* P = psm;
  double* lam = psm + N * PPITCH;            // [128]
  double* xch = lam + N;                     // [128] interface value received from the partner
  // mbarriers: bar[0] = interface values arrived (phase 3), bar[1] = v(z = 63) arrived (rank 1)
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(xch + N), bar1 = bar0 + 8;
  const int rank = (int)cluster.block_rank();
  const long plane = blockIdx.x >> 1;        // field * 128 + a
  const int a = (int)(plane & (N - 1));
  double* gp = u + (size_t)plane * NN + (size_t)rank * PHC;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  FACR_MARK(0);
  if (t == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    mbar_fence_init();
  }
  cluster_arrive_relaxed();                  // (waited for before the first remote store)
  for (int i = t; i < N; i += PTHR) lam[i] = lam_g[i];
  {
    const unsigned sb = (unsigned)__cvta_generic_to_shared(P);
#if !PLANE_SOL_NOLOAD
#pragma unroll 16
    for (int e = t; e < N * PHC; e += PTHR) {
      // a warp covers 32 consecutive z of one row: lanes 0-15 the odd z (kept columns), lanes
      // 16-31 the even z (eliminated columns), so each half-warp hits 16 distinct bank pairs
      const int r = e >> 6, c = ((e >> 5) & 1) * 16 + (e & 15) + ((e & 16) ? 32 : 0);
      const int z = 2 * (c & 31) + ((e & 16) ? 0 : 1);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + 8u * (unsigned)(r * PPITCH + c)),
                   "l"(gp + (size_t)r * N + z));
    }
#endif
    if (rank == 0)   // z = 64 (the partner's first column; an L2 hit, the partner reads it too)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + 8u * (unsigned)(t * PPITCH + PHC)),
                   "l"(gp + (size_t)t * N + PHC));
    else
      P[t * PPITCH + PHC] = 0.0;
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  FACR_MARK(1);
  const double hsa = h2 * (inv_dt + lam[a]);
  const double beta = 4.0 + hsa;
  // (1) r_i = gs (β g_z[y] - g_z[y-1] - g_z[y+1] + g_{z-1}[y] + g_{z+1}[y]),  z = 2i + 1,  i = lane
  if (!PLANE_SOL_NOP1) {
    const int y0 = 32 * warp;
    const double* gk = P + lane;             // kept column i
    const double* gl = P + 32 + lane;        // eliminated j = i   (z - 1)
    const double* gr = P + 33 + lane;        // eliminated j = i+1 (z + 1; col 64 for i = 31)
    double rr[32];
    double prev = y0 > 0 ? gk[(y0 - 1) * PPITCH] : 0.0, cur = gk[y0 * PPITCH];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int y = y0 + j;
      const double nxt = y + 1 < N ? gk[(y + 1) * PPITCH] : 0.0;
      rr[j] = gs * (fma(beta, cur, -(prev + nxt)) + (gl[y * PPITCH] + gr[y * PPITCH]));
      prev = cur;
      cur = nxt;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) P[(y0 + j) * PPITCH + lane] = rr[j];
    if (rank == 0) P[t * PPITCH + PHC] = 0.0;   // ghost z = -1 for phase 5
  }
  __syncthreads();
  FACR_MARK(2);
#if PLANE_YDST_INLINE
  plane_ydst<true>(P);
#else
  if (!PLANE_SOL_NOXF) plane_ydst_call<true>(P);
#endif
  __syncthreads();
  FACR_MARK(3);
  // (3) reduced system per y-mode row b: -u_{i-1} + d u_i - u_{i+1} = ys r̂_i over the 64 kept z,
  //     d = τ² - 2 = μ + 1/μ with μ = μ_τ², last global row d + 1.
  {
    const int b = t;
    double* row = P + b * PPITCH;            // kept entry i at row[i]
    constexpr int M = PHC / 2;
    constexpr double ys = 2.0 / (N + 1);
    const double hs = h2 * ((inv_dt + lam[a]) + lam[b]);
    const double mut = 2.0 / ((2.0 + hs) + sqrt(hs * (hs + 4.0)));
    const double mu = mut * mut;
    double v[M];                                           // the row, in registers until the end
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = ys * row[i];
    if (!PLANE_SOL_NOP3) {
#pragma unroll
      for (int i = 1; i < M; ++i) v[i] = fma(mu, v[i - 1], v[i]);
#pragma unroll
      for (int i = M - 2; i >= 0; --i) v[i] = fma(mu, v[i + 1], v[i]);
    }
    double muM = mu;                                       // μ^M, M = 32
#pragma unroll
    for (int q = 0; q < 5; ++q) muM *= muM;
    const double mu2 = mu * mu;
    const double mu2M1 = muM * muM * mu;                   // μ^{2M+1}
    const double den = 1.0 - mu2M1 * mu;                   // 1 - μ^{2M+2}
    const double c2 = mu2 * v[0] / den;
    const double a31 = fma(mu, v[M - 1], -c2 * (muM - muM * mu2));     // local Dirichlet x_{M-1}
    const double a0 = fma(mu, v[0], -c2 * (mu - mu2M1));              // local Dirichlet x_0
    const double gL0 = muM * (1.0 - mu2) / den;            // g_L[0]   (g_L = T^{-1} e_{M-1})
    const double gam0 = mu * (1.0 - muM * muM) / den;      // g_L[M-1] = g_R[0]
    const double sm = 1.0 / (1.0 + gam0);
    const double mine = rank == 0 ? a31 : a0 - gL0 * a31 * sm;   // rank 1: last row +1 (Sherman–Morrison)
    if (b == 0) mbar_expect_tx(bar0, N * sizeof(double));
    cluster_wait();                          // the partner's mbarriers are initialised
    st_async(mapa((unsigned)__cvta_generic_to_shared(xch + b), rank ^ 1), mine, mapa(bar0, rank ^ 1));
    mbar_wait(bar0, 0);
    const double other = xch[b];
    const double x31 = rank == 0 ? mine : other, x32 = rank == 0 ? other : mine;
    const double gam1 = gam0 - gL0 * gL0 * sm;             // right half's response at its first entry
    const double u31 = (x31 + x32 * gam0) / (1.0 - gam0 * gam1);
    const double u32 = x32 + u31 * gam1;
    // u_i = μ z_i + A (μ^{i+1} - μ^{2M+1-i}) + B (μ^{M-i} - μ^{M+i+2})
    const double A = rank == 0 ? -c2 : u31 / den - c2;
    const double B = rank == 0 ? u32 / den : -(a31 + u31 * gL0) * sm / den;
    const double imu = 1.0 / mu;
    if (PLANE_SOL_NOP3) {
#pragma unroll
      for (int i = 0; i < M; ++i) row[i] = v[i] + A + B;
    } else {
    double pa = mu, pb = mu2M1;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      v[i] = fma(mu, v[i], A * (pa - pb));
      pa *= mu;
      pb *= imu;
    }
    double ga = mu, gb = mu2M1;                            // at i = M-1
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
      row[i] = fma(B, ga - gb, v[i]);
      ga *= mu;
      gb *= imu;
    }
    }
  }
  __syncthreads();
  FACR_MARK(4);
#if PLANE_YDST_INLINE
  plane_ydst<true>(P);
#else
  if (!PLANE_SOL_NOXF) plane_ydst_call<true>(P);
#endif
  __syncthreads();
  FACR_MARK(5);
  // rank 0 pushes v(z = 63) into rank 1's neighbour column (rank 1 finished reading its ghost
  // column in phase 1 before the interface barrier above); rank 1 waits for it, rank 0 only
  // before exiting.
  if (rank == 0) {
    st_async(mapa((unsigned)__cvta_generic_to_shared(P + t * PPITCH + PHC), 1), P[t * PPITCH + 31], mapa(bar1, 1));
  } else {
    if (t == 0) mbar_expect_tx(bar1, N * sizeof(double));
    mbar_wait(bar1, 0);
  }
  FACR_MARK(6);
  // (5) eliminated column j = 16 (warp/2) + 2 (lane%8) + warp%2, row segment s = lane/8:
  //     [0,33) [33,64) [64,97) [97,128); a half-warp holds 8 columns of one parity x 2 segments
  //     whose start rows are ≡ 0, 1 mod 16: 16 distinct 8-byte bank pairs
  if (!PLANE_SOL_NOP5) {
    const int j = 16 * (warp >> 1) + 2 * (lane & 7) + (warp & 1), s = lane >> 3;
    const int kb = (s >> 1) * 64 + (s & 1) * 33, L = (s & 1) ? 31 : 33;
    const double muy = 2.0 / (beta + sqrt((beta - 2.0) * (beta + 2.0)));
    const double imu = 1.0 / muy, mu2 = muy * muy;
    double* col = P + kb * PPITCH + 32 + j;
    const double* vl = P + kb * PPITCH + (j == 0 ? PHC : j - 1);   // v at z - 1
    const double* vr = P + kb * PPITCH + j;                        // v at z + 1
    // the segment stays in registers (x[q], q < L <= 33) from the first load to the final store
    // S1: local forward sweep ŷ_k = r_k + μ ŷ_{k-1},  r = gs g + v_{z-1} + v_{z+1}
    double x[33];
#pragma unroll
    for (int q = 0; q < 33; ++q)
      x[q] = q < L ? fma(gs, col[q * PPITCH], vl[q * PPITCH] + vr[q * PPITCH]) : 0.0;
#pragma unroll
    for (int q = 1; q < 33; ++q) x[q] = fma(muy, x[q - 1], x[q]);
    const double yv = (s & 1) ? x[30] : x[32];
    const int base = lane & 7;
#if PLANE_P5_MERGED
    // the powers of μ this phase needs, from 5 squarings and a few products (all of them shrink with the
    // exponent: an underflow to 0 only drops terms that are themselves negligible, as with ipow128)
    const double m4 = mu2 * mu2, m8 = m4 * m4, m16 = m8 * m8, m32 = m16 * m16;
    const double mu31 = ((m16 * m8) * (m4 * mu2)) * muy, mu33 = m32 * muy;
    const double m64 = m32 * m32, m128 = m64 * m64, m256 = m128 * m128;
#else
    const double mu33 = ipow128(muy, 33), mu31 = ipow128(muy, 31);
#endif
    const double Y0 = __shfl_sync(0xffffffffu, yv, base), Y1 = __shfl_sync(0xffffffffu, yv, base + 8),
                 Y2 = __shfl_sync(0xffffffffu, yv, base + 16);
    // incoming true y_{kb-1}: segment lengths 33, 31, 33
    const double c1 = Y0, c2f = fma(mu31, c1, Y1), c3 = fma(mu33, c2f, Y2);
    const double cin = s == 0 ? 0.0 : s == 1 ? c1 : s == 2 ? c2f : c3;
    // S2: local backward sweep ẑ_k = ŷ_k + μ ẑ_{k+1} (entries q >= L are zero, and stay so)
    if (s & 1) {
      x[31] = x[32] = 0.0;
    }
#pragma unroll
    for (int q = 31; q >= 0; --q) x[q] = fma(muy, x[q + 1], x[q]);
    // true z_k = ẑ_k + cin ζ_k + μ^{ke-k} Zr,  ζ_k = (μ^{k-kb+1} - μ^{2ke-kb+1-k}) / (1 - μ²)
    const double i1m = 1.0 / (1.0 - mu2);
    const double muL = s & 1 ? mu31 : mu33;
    const double tb = fma(cin, muy * (1.0 - muL * muL) * i1m, x[0]);   // ẑ_kb + cin ζ_kb
    const double T0 = __shfl_sync(0xffffffffu, tb, base), T1 = __shfl_sync(0xffffffffu, tb, base + 8),
                 T2 = __shfl_sync(0xffffffffu, tb, base + 16), T3 = __shfl_sync(0xffffffffu, tb, base + 24);
    const double Z3 = T3, Z2 = fma(mu33, Z3, T2), Z1 = fma(mu31, Z2, T1), Z0 = fma(mu33, Z1, T0);
    const double Zr = s == 0 ? Z1 : s == 1 ? Z2 : s == 2 ? Z3 : 0.0;   // true z at ke
    // S3 (ascending): w_k = μ (ẑ_k + cin ζ_k) - c2 (μ^{k+1} - μ^{2n+1-k}),  c2 = μ² z_0 / (1 - μ^{2n+2})
#if PLANE_P5_MERGED
    // the four running powers of the unmerged form pair up: μ^{q+1} and μ^{kb+1+q} are both ∝ μ^q, μ^{2L+1-q}
    // and μ^{2n+1-kb-q} both ∝ μ^{-q}, so  w_q = μ x_q + a_q + b_q  with
    //   a_q = (ci μ² - c2 μ^{kb+1}) μ^q,   b_q = (c2 μ^{2n+1-kb} - ci μ^{2L+2}) μ^{-q}
    // (same walking directions as before: a shrinks, b grows from a start that is negligible when tiny)
    const double c2 = mu2 * Z0 / (1.0 - m256 * mu2);
    const double ci = cin * i1m;
    const double mu34 = mu33 * muy;
    const double pkb = s == 0 ? muy : s == 1 ? mu34 : s == 2 ? m64 * muy : m64 * mu34;          // μ^{kb+1}
    const double pnk = s == 0 ? m256 * muy : s == 1 ? (m128 * m64) * m32 : s == 2 ? (m128 * m64) * muy
                                                                                   : m128 * m32;   // μ^{2n+1-kb}
    const double p2l = (s & 1) ? m64 : m64 * m4;                                                   // μ^{2L+2}
    double aq = fma(ci, mu2, -c2 * pkb), bq = fma(c2, pnk, -ci * p2l);
#pragma unroll
    for (int q = 0; q < 33; ++q) {
      x[q] = fma(muy, x[q], aq + bq);
      aq *= muy;
      bq *= imu;
    }
#else
    const double c2 = mu2 * Z0 / (1.0 - ipow128(muy, 2 * N + 2));
    const double ci = cin * i1m;
    double p1 = muy, p2 = ipow128(muy, 2 * L + 1);                // μ^{k-kb+1}, μ^{2ke-kb+1-k}
    double pa = ipow128(muy, kb + 1), pb = ipow128(muy, 2 * N + 1 - kb);
#pragma unroll
    for (int q = 0; q < 33; ++q) {
      x[q] = fma(muy, fma(ci, p1 - p2, x[q]), -c2 * (pa - pb));
      p1 *= muy;
      p2 *= imu;
      pa *= muy;
      pb *= imu;
    }
#endif
    // S4 (descending): + μ^{ke-k+1} Zr, then the single store of the segment
    double pr = mu2 * Zr;                                          // Zr = 0 for the last segment
    if (s & 1) {
#pragma unroll
      for (int q = 30; q >= 0; --q) {
        col[q * PPITCH] = x[q] + pr;
        pr *= muy;
      }
    } else {
#pragma unroll
      for (int q = 32; q >= 0; --q) {
        col[q * PPITCH] = x[q] + pr;
        pr *= muy;
      }
    }
  }
  __syncthreads();
  FACR_MARK(7);
  PLANE_UNROLL(PLANE_STORE_UNROLL)
  for (int e = t; e < (PLANE_SOL_NOSTORE ? 0 : N * PHC); e += PTHR) {   // same lane -> (column, z) map as the load
    const int r = e >> 6, c = ((e >> 5) & 1) * 16 + (e & 15) + ((e & 16) ? 32 : 0);
    const int z = 2 * (c & 31) + ((e & 16) ? 0 : 1);
#if PLANE_STORE_CS
    __stcs(gp + (size_t)r * N + z, P[r * PPITCH + c]);
#else
    __stcg(gp + (size_t)r * N + z, P[r * PPITCH + c]);
#endif
  }
  FACR_MARK(8);
  // no exit barrier: each CTA has consumed every remote store aimed at it (its mbarrier waits), and
  // issues none after its partner's last wait
}

unsigned long long g_tables_ready = 0;   // bit d: constant tables uploaded on device d

}  // namespace

// Per-plan A-fragment table (device memory owned by the plan).
cudaError_t dst128_atab(double** tab) {
  cudaError_t e = cudaMalloc(tab, ATAB * sizeof(double));
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(1);
  pfa_atab_kernel<<<ATAB / 32, 32>>>(*tab);
  return cudaGetLastError();
}

cudaError_t dst128_init() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && (g_tables_ready >> dev) & 1ull) return cudaSuccess;
  const Tables t = make_tables();
  for (int r = 0; r < N; ++r)
    if (t.slot[r] == 255) return cudaErrorInvalidValue;   // the CRT map must cover every row
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c_slot, t.slot, sizeof(t.slot))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_usign, t.usign, sizeof(t.usign))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_wsign, t.wsign, sizeof(t.wsign))) != cudaSuccess) return e;
  double s43[43], c43[43];
  for (int m = 0; m < 43; ++m) {   // long double evaluation, rounded once to double
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / 43.0L;
    s43[m] = (double)sinl(a);
    c43[m] = (double)(0.866025403784438646763723170752936183L * cosl(a));
  }
  if ((e = cudaMemcpyToSymbol(c_s43, s43, sizeof(s43))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_c43, c43, sizeof(c43))) != cudaSuccess) return e;
  if (dev < 64) g_tables_ready |= 1ull << dev;
  return cudaSuccess;
}

// One DST-I pass (scale 1) along x (pass 0) or y (pass 1) of nfields n=128 fields; out may == in.
cudaError_t dst128_pass(int pass, const double* in, double* out, int nfields, const double* atab, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static const int use_dmma = [] {
    const char* v = getenv("DPM_DST128_DMMA");
    return v && atoi(v) == 1;
  }();
  if (!use_dmma) {
    const size_t smem = 7 * (IN_SIZE + RAW_SIZE) * sizeof(double);
    static const int minb = [] {
      const char* v = getenv("DPM_DST128F_MINB");
      return v && atoi(v) == 2 ? 2 : 1;
    }();
    auto kf = minb == 1 ? (pass == 0 ? dst128f_kernel<0, 1> : dst128f_kernel<1, 1>)
                        : (pass == 0 ? dst128f_kernel<0, 2> : dst128f_kernel<1, 2>);
    cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, 224, smem);
    const long warps = (long)nfields * (NN / 16);
    const int grid = (int)std::min<long>((warps + 6) / 7, (long)sms * std::max(1, occ));
    DPM_COUNT_LAUNCH(1);
    kf<<<grid, 224, smem, s>>>(in, out, nfields, nullptr, nullptr, 0);
    return cudaGetLastError();
  }
  const size_t smem = 2 * (size_t)TILE * sizeof(double);
  auto k = pass == 0 ? dst128_pass_kernel<0> : dst128_pass_kernel<1>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTHR, smem);
  const long ntiles = (long)nfields * (NN / TC);
  const int grid = (int)std::min<long>(ntiles, (long)sms * std::max(1, occ));
  DPM_COUNT_LAUNCH(1);
  k<<<grid, NTHR, smem, s>>>(in, out, nfields, atab);
  return cudaGetLastError();
}

// forward x pass of the fused BEP build (MODE 1 above): same grid as the dense pass.
cudaError_t dst128_xpass_sparse(double* out, int nfields, const uint32_t* tab, const double* vals, int64_t ldv,
                                cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = 7 * (IN_SIZE + RAW_SIZE) * sizeof(double);
  auto kf = dst128f_kernel<0, 1, 1>;
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, 224, smem);
  const long warps = (long)nfields * (NN / 16);
  const int grid = (int)std::min<long>((warps + 6) / 7, (long)sms * std::max(1, occ));
  DPM_COUNT_LAUNCH(1);
  kf<<<grid, 224, smem, s>>>(nullptr, out, nfields, tab, vals, ldv);
  return cudaGetLastError();
}

// Fused y-DST / z-tridiagonal / inverse y-DST over nfields n = 128 fields (in place), after the x pass.
// xscale = 2/(n+1) (x transform pair) and rscale = xscale² h²; DPM_PLANE_FACR=0 selects the
// full-transform plane kernel instead of FACR(1).
cudaError_t plane128_pass(double* u, int nfields, const double* lam, double inv_dt, double h2, double rscale,
                          cudaStream_t s) {
  static const bool facr = [] {
    const char* v = getenv("DPM_PLANE_FACR");
    return !(v && atoi(v) == 0);
  }();
  auto k = facr ? plane128_facr_kernel : plane128_kernel;
  const double arg = facr ? rscale * (N + 1) / 2.0 : rscale;   // FACR: x normalisation · h² only
  const size_t smem = ((size_t)N * PPITCH + 2 * N + 2) * sizeof(double);   // + 2 mbarriers (FACR)
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long ctas = 2L * nfields * N;
  if (ctas > 2147483647L) return cudaErrorInvalidValue;
  DPM_COUNT_LAUNCH(1);
  k<<<(unsigned)ctas, PTHR, smem, s>>>(u, lam, inv_dt, h2, arg);
  return cudaGetLastError();
}

#if FACR_PHASE_TIMING
extern "C" int dpm_debug_facr_phases(unsigned long long* host, int nctas) {
  const int n = nctas < FACR_TCTAS ? nctas : FACR_TCTAS;
  return (int)cudaMemcpyFromSymbol(host, g_facr_ph, (size_t)n * FACR_TPH * sizeof(unsigned long long));
}
#endif
