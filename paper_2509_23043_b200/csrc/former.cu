// former.cu -- IsingFormer proposal model on the device (Appendix F;
// the reference's proj/src/generator.cpp:1 is a placeholder).  Inference only: forward logits,
// exact log q (the MH-corrected acceptance of tapt_inject_proposals consumes it) and ancestral
// sampling from counter-based splitmix64 streams.  Host side: configuration, seeded parameter
// initialisation and the ISFW1 checkpoint format.
//
// Kernel ("row engine"): a CTA of 256 threads advances a block of 32 ROWS through the decoder.
// A row is one (sequence, position).  Forward/log_prob: the rows are 32 consecutive positions of
// one sequence.  Sampling: the rows are 32 sequences at the same position.  Per row the layer
// computes LN1 -> QKV (K, V appended to the row's cache in HBM) -> causal attention over the
// row's cached keys (one warp per (row, head), online softmax over 32-key chunks, each chunk's
// K and V loads issued together) -> out-projection + residual -> LN2 ->
// FFN (GELU) + residual.  The dense products read fp32 weights from global memory (L1/L2
// resident, 267 KB) with one column per lane and 8 rows per thread, so every weight load is
// shared by 8 rows.  Sampling is bound by the K/V cache reads: sum over t of t x 2 layers x
// (K + V) x 64 x 4 B per sequence.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "tc.cuh"
#include "tapt/errors.hpp"
#include "tapt/rng.hpp"
#include "tapt_gpu.h"

namespace tapt_host {
void set_last_error(const std::string& m);
void note_launches(unsigned n);
}  // namespace tapt_host

namespace tapt_former_dev {

constexpr int D = 64, F = 128, DH = 32, NT = 256, kMaxL = 16;

struct LayerOff {
    int ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_1, b_1, w_2, b_2;
};

struct FArgs {
    const float* W;  // parameters (canonical ISFW1 order)
    int tok_emb, beta_w, beta_b, lnf_g, lnf_b, head_w, head_b;
    LayerOff lay[kMaxL];
    int L, fb;
    const float* pos;  // [max_len][D] sinusoidal positions
    int T, n_prefix, B;
    void* cache;   // [slots][L][T][2][D]: K then V of every cached position (float or bf16, KVT below)
    const uint8_t* tokens;     // forward: [B][T]; sample: prefix [B][n_prefix]
    const double* betas;       // [B]
    float* logits;             // forward: [B][T] (nullable)
    double* log_q;             // [B]
    uint8_t* tok_out;          // sample: [B][T]
    const uint64_t* streams;   // sample: [B]
};

template <int RB>
struct Smem {
    float X[RB][D];   // residual stream
    float A[RB][D];   // LayerNorm output
    float Q[RB][D];   // queries
    float O[RB][D];   // attention output
    float Fh[RB][F];  // FFN hidden
    float Eb[RB][D];  // beta embedding of each row's sequence
    float z[RB];      // logits
    int t[RB];        // position of each row
    int slot[RB];     // cache slot of each row
    int valid[RB];
    int tokprev[RB];
    double lq[RB];
};

// K/V chunk staged by the forward kernel (rows share one sequence's keys): 32 keys x (K | V) of
// 64 dims, row stride 65 so that lanes reading different keys fall in different banks.
struct KVChunk {
    float K[32][2 * 32 + 1];
    float V[32][2 * 32 + 1];
    float4 P[NT / 32][8];  // per warp: the 32 key probabilities of the current task (float4-read)
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}

// LayerNorm of every row (eps 1e-5): warp w handles rows w, w+8, ...; lane holds 2 values.
template <int RB>
__device__ void rows_ln(const float (&X)[RB][D], float (&A)[RB][D], const float* g, const float* b) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int r = w; r < RB; r += NT / 32) {
        const float x0 = X[r][lane], x1 = X[r][lane + 32];
        const float mu = warp_sum(x0 + x1) * (1.0f / D);
        const float d0 = x0 - mu, d1 = x1 - mu;
        const float var = warp_sum(d0 * d0 + d1 * d1) * (1.0f / D);
        const float inv = rsqrtf(var + 1e-5f);
        A[r][lane] = d0 * inv * __ldg(g + lane) + __ldg(b + lane);
        A[r][lane + 32] = d1 * inv * __ldg(g + lane + 32) + __ldg(b + lane + 32);
    }
}

__device__ __forceinline__ float gelu(float x) {
    return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}

// Out[r][c] = sum_k In[r][k] W[k][c] + b[c] for the RB rows: lane group (tid & 63) owns
// columns c0 + 64j, tid >> 6 selects rows rg + 4i; A is read 4 k at a time (LDS.128,
// broadcast within a warp).  EPI: 0 store, 1 residual add into Out, 2 GELU then store.
template <int RB, int N, int K, int EPI>
__device__ void rows_gemm(const float* In, const float* W, const float* bias, float* Out) {
    constexpr int NC = N / 64, NR = RB / 4;
    const int c0 = threadIdx.x & 63, rg = threadIdx.x >> 6;
    float acc[NR][NC];
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[i][j] = 0.f;
#pragma unroll 2
    for (int k = 0; k < K; k += 4) {
        float w[4][NC];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int j = 0; j < NC; ++j) w[kk][j] = __ldg(W + (size_t)(k + kk) * N + c0 + 64 * j);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const float4 a = *reinterpret_cast<const float4*>(In + (rg + 4 * i) * K + k);
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                acc[i][j] = fmaf(a.x, w[0][j], acc[i][j]);
                acc[i][j] = fmaf(a.y, w[1][j], acc[i][j]);
                acc[i][j] = fmaf(a.z, w[2][j], acc[i][j]);
                acc[i][j] = fmaf(a.w, w[3][j], acc[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const int r = rg + 4 * i, c = c0 + 64 * j;
            const float v = acc[i][j] + __ldg(bias + c);
            if constexpr (EPI == 0) Out[r * N + c] = v;
            if constexpr (EPI == 1) Out[r * N + c] += v;
            if constexpr (EPI == 2) Out[r * N + c] = gelu(v);
        }
}

// K/V cache element: float (default) or bf16 (opt-in: half the bytes of the sampling-bound stream;
// the attention math stays fp32).  ld4 reads 4 consecutive elements as a float4.
template <class KT>
struct KVT;
template <>
struct KVT<float> {
    static __device__ __forceinline__ float4 ld4(const void* base, size_t i) {
        return *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + i);
    }
    static __device__ __forceinline__ void st(void* base, size_t i, float v) { reinterpret_cast<float*>(base)[i] = v; }
    static __device__ __forceinline__ void ld8(const void* base, size_t i, float4& a, float4& b) {
        a = ld4(base, i);
        b = ld4(base, i + 4);
    }
};
template <>
struct KVT<__nv_bfloat16> {
    static __device__ __forceinline__ float4 ld4(const void* base, size_t i) {
        const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(base) + i);
        return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                           __uint_as_float(u.y & 0xFFFF0000u));
    }
    static __device__ __forceinline__ void st(void* base, size_t i, float v) {
        reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
    }
    static __device__ __forceinline__ void ld8(const void* base, size_t i, float4& a, float4& b) {  // one 16-B load
        const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + i);
        a = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                        __uint_as_float(u.y & 0xFFFF0000u));
        b = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u), __uint_as_float(u.w << 16),
                        __uint_as_float(u.w & 0xFFFF0000u));
    }
};

// QKV projection: Q to shared memory, K and V appended to each valid row's cache.
template <int RB, class KT>
__device__ void rows_qkv(Smem<RB>& s, const FArgs& a, int l) {
    constexpr int NR = RB / 4;
    const LayerOff& o = a.lay[l];
    const float* W = a.W + o.w_qkv;
    const float* bias = a.W + o.b_qkv;
    const int c0 = threadIdx.x & 63, rg = threadIdx.x >> 6;
    float acc[NR][3];
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) acc[i][j] = 0.f;
#pragma unroll 2
    for (int k = 0; k < D; k += 4) {
        float w[4][3];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int j = 0; j < 3; ++j) w[kk][j] = __ldg(W + (size_t)(k + kk) * 3 * D + c0 + 64 * j);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const float4 x = *reinterpret_cast<const float4*>(&s.A[rg + 4 * i][k]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                acc[i][j] = fmaf(x.x, w[0][j], acc[i][j]);
                acc[i][j] = fmaf(x.y, w[1][j], acc[i][j]);
                acc[i][j] = fmaf(x.z, w[2][j], acc[i][j]);
                acc[i][j] = fmaf(x.w, w[3][j], acc[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const int r = rg + 4 * i;
        s.Q[r][c0] = acc[i][0] + __ldg(bias + c0);
        if (s.valid[r]) {
            const size_t kv = ((((size_t)s.slot[r] * a.L + l) * a.T + s.t[r]) * 2) * D;
            KVT<KT>::st(a.cache, kv + c0, acc[i][1] + __ldg(bias + D + c0));
            KVT<KT>::st(a.cache, kv + D + c0, acc[i][2] + __ldg(bias + 2 * D + c0));
        }
    }
}

// Causal attention of every valid row over its cached positions 0..t (2 heads of 32): one
// warp per (row, head), online softmax over 32-key chunks.  Per chunk every lane issues all of
// its loads up front -- its key's K row (8 x float4) and a float4 slice of 8 V rows (keys
// c + 4i + lane/8, dims 4*(lane%8)..+3) -- so a chunk costs one memory round trip; the lanes
// sharing a dimension slice are reduced once per task.
template <int RB, class KT>
__device__ void rows_attention(Smem<RB>& s, const FArgs& a, int l, int H) {
    // V slice per lane: fp32 4 dims of 8 keys (8 lanes per key); bf16 8 dims of 4 keys (4 lanes per
    // key) so that every load is 16 bytes
    constexpr bool W8 = sizeof(KT) == 2;
    constexpr int VD = W8 ? 8 : 4, LPK = DH / VD, KPP = 32 / LPK, NP = 32 / KPP;  // dims, lanes/key, keys/pass, passes
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int kq = lane / LPK, dq = VD * (lane % LPK);
    const float scale = rsqrtf((float)DH);
    for (int task = w; task < RB * H; task += NT / 32) {
        const int r = task / H, h = task - r * H;
        if (!s.valid[r]) {
            s.O[r][h * DH + lane] = 0.f;
            continue;
        }
        const int tr = s.t[r];
        const size_t base = (((size_t)s.slot[r] * a.L + l) * a.T) * 2 * D + h * DH;
        const float4* q4 = reinterpret_cast<const float4*>(&s.Q[r][h * DH]);
        float m = -INFINITY, lsum = 0.f;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f), o2 = o;
        for (int c = 0; c <= tr; c += 32) {
            const int j = c + lane;
            float4 kk[DH / 4], vv[NP], vv2[NP];
#pragma unroll
            for (int q = 0; q < DH / 4; q += 2) {
                if (j <= tr) {
                    KVT<KT>::ld8(a.cache, base + (size_t)j * 2 * D + 4 * q, kk[q], kk[q + 1]);
                } else {
                    kk[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    kk[q + 1] = kk[q];
                }
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const int key = c + KPP * i + kq;
                vv[i] = vv2[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (key <= tr) {
                    if constexpr (W8)
                        KVT<KT>::ld8(a.cache, base + (size_t)key * 2 * D + D + dq, vv[i], vv2[i]);
                    else
                        vv[i] = KVT<KT>::ld4(a.cache, base + (size_t)key * 2 * D + D + dq);
                }
            }
            float acc = 0.f;
#pragma unroll
            for (int q = 0; q < DH / 4; ++q) {
                const float4 qq = q4[q];
                acc = fmaf(qq.x, kk[q].x, acc);
                acc = fmaf(qq.y, kk[q].y, acc);
                acc = fmaf(qq.z, kk[q].z, acc);
                acc = fmaf(qq.w, kk[q].w, acc);
            }
            const float sc = j <= tr ? acc * scale : -INFINITY;
            const float mn = fmaxf(m, warp_max(sc));
            const float corr = __expf(m - mn);  // m = -inf on the first chunk -> 0
            const float p = j <= tr ? __expf(sc - mn) : 0.f;
            lsum = lsum * corr + warp_sum(p);
            o.x *= corr;
            o.y *= corr;
            o.z *= corr;
            o.w *= corr;
            if constexpr (W8) {
                o2.x *= corr;
                o2.y *= corr;
                o2.z *= corr;
                o2.w *= corr;
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const float pk = __shfl_sync(0xFFFFFFFFu, p, KPP * i + kq);
                o.x = fmaf(pk, vv[i].x, o.x);
                o.y = fmaf(pk, vv[i].y, o.y);
                o.z = fmaf(pk, vv[i].z, o.z);
                o.w = fmaf(pk, vv[i].w, o.w);
                if constexpr (W8) {
                    o2.x = fmaf(pk, vv2[i].x, o2.x);
                    o2.y = fmaf(pk, vv2[i].y, o2.y);
                    o2.z = fmaf(pk, vv2[i].z, o2.z);
                    o2.w = fmaf(pk, vv2[i].w, o2.w);
                }
            }
            m = mn;
        }
#pragma unroll
        for (int x = LPK; x <= 16; x <<= 1) {  // lanes sharing a dimension slice
            o.x += __shfl_xor_sync(0xFFFFFFFFu, o.x, x);
            o.y += __shfl_xor_sync(0xFFFFFFFFu, o.y, x);
            o.z += __shfl_xor_sync(0xFFFFFFFFu, o.z, x);
            o.w += __shfl_xor_sync(0xFFFFFFFFu, o.w, x);
            if constexpr (W8) {
                o2.x += __shfl_xor_sync(0xFFFFFFFFu, o2.x, x);
                o2.y += __shfl_xor_sync(0xFFFFFFFFu, o2.y, x);
                o2.z += __shfl_xor_sync(0xFFFFFFFFu, o2.z, x);
                o2.w += __shfl_xor_sync(0xFFFFFFFFu, o2.w, x);
            }
        }
        if (lane < LPK) {
            const float inv = 1.f / lsum;
            *reinterpret_cast<float4*>(&s.O[r][h * DH + dq]) = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
            if constexpr (W8)
                *reinterpret_cast<float4*>(&s.O[r][h * DH + dq + 4]) =
                    make_float4(o2.x * inv, o2.y * inv, o2.z * inv, o2.w * inv);
        }
    }
}

// Causal attention for the forward pass, where the 32 rows are consecutive positions of ONE
// sequence: every 32-key chunk of the cache is staged in shared memory once per row block and
// read by all (row, head) tasks (flash-attention style).  Warp w owns tasks w, w+8, ... and
// keeps their online-softmax state in registers across chunks.
template <int RB, class KT>
__device__ void rows_attention_fwd(Smem<RB>& s, KVChunk& kv, const FArgs& a, int l) {
    constexpr int H = D / DH, NTASK = RB * H / (NT / 32);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float scale = rsqrtf((float)DH);
    const size_t base = (((size_t)s.slot[0] * a.L + l) * a.T) * 2 * D;
    int tmax = -1;
    for (int r = 0; r < RB; ++r)
        if (s.valid[r]) tmax = max(tmax, s.t[r]);
    float m[NTASK], lsum[NTASK], o[NTASK];
#pragma unroll
    for (int k = 0; k < NTASK; ++k) {
        m[k] = -INFINITY;
        lsum[k] = 0.f;
        o[k] = 0.f;
    }
    for (int c = 0; c <= tmax; c += 32) {
        __syncthreads();  // previous chunk fully consumed
        for (int e = threadIdx.x; e < 32 * 2 * D / 4; e += NT) {  // 32 keys x (K 64 | V 64), float4
            const int key = e / (2 * D / 4), q4 = e - key * (2 * D / 4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c + key <= tmax) v = KVT<KT>::ld4(a.cache, base + (size_t)(c + key) * 2 * D + 4 * q4);
            float* dst = q4 < D / 4 ? &kv.K[key][4 * q4] : &kv.V[key][4 * q4 - D];
            dst[0] = v.x;
            dst[1] = v.y;
            dst[2] = v.z;
            dst[3] = v.w;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NTASK; ++k) {
            const int task = w + k * (NT / 32), r = task / H, h = task - r * H;
            const int tr = s.t[r];
            if (!s.valid[r] || c > tr) continue;  // warp-uniform
            const int j = c + lane;
            float acc = 0.f;
#pragma unroll 8
            for (int d = 0; d < DH; ++d) acc = fmaf(s.Q[r][h * DH + d], kv.K[lane][h * DH + d], acc);
            const float sc = j <= tr ? acc * scale : -INFINITY;
            const float mn = fmaxf(m[k], warp_max(sc));
            const float corr = __expf(m[k] - mn);
            const float p = j <= tr ? __expf(sc - mn) : 0.f;
            lsum[k] = lsum[k] * corr + warp_sum(p);
            float oo = o[k] * corr;
            reinterpret_cast<float*>(kv.P[w])[lane] = p;  // broadcast through shared memory, not 32 shuffles
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float4 pq = kv.P[w][q];
                oo = fmaf(pq.x, kv.V[4 * q + 0][h * DH + lane], oo);
                oo = fmaf(pq.y, kv.V[4 * q + 1][h * DH + lane], oo);
                oo = fmaf(pq.z, kv.V[4 * q + 2][h * DH + lane], oo);
                oo = fmaf(pq.w, kv.V[4 * q + 3][h * DH + lane], oo);
            }
            __syncwarp();
            o[k] = oo;
            m[k] = mn;
        }
    }
#pragma unroll
    for (int k = 0; k < NTASK; ++k) {
        const int task = w + k * (NT / 32), r = task / H, h = task - r * H;
        s.O[r][h * DH + lane] = s.valid[r] ? o[k] / lsum[k] : 0.f;
    }
}

// All decoder layers + final LayerNorm + head for the current row block; logits in s.z.
template <int RB, class KT>
__device__ void rows_forward(Smem<RB>& s, const FArgs& a, KVChunk* kv = nullptr) {
    const int H = D / DH;
    for (int l = 0; l < a.L; ++l) {
        const LayerOff& o = a.lay[l];
        rows_ln(s.X, s.A, a.W + o.ln1_g, a.W + o.ln1_b);
        __syncthreads();
        rows_qkv<RB, KT>(s, a, l);
        __syncthreads();
        if constexpr (RB == 32) {
            if (kv)
                rows_attention_fwd<RB, KT>(s, *kv, a, l);
            else
                rows_attention<RB, KT>(s, a, l, H);
        } else {
            rows_attention<RB, KT>(s, a, l, H);
        }
        __syncthreads();
        rows_gemm<RB, D, D, 1>(&s.O[0][0], a.W + o.w_o, a.W + o.b_o, &s.X[0][0]);
        __syncthreads();
        rows_ln(s.X, s.A, a.W + o.ln2_g, a.W + o.ln2_b);
        __syncthreads();
        rows_gemm<RB, F, D, 2>(&s.A[0][0], a.W + o.w_1, a.W + o.b_1, &s.Fh[0][0]);
        __syncthreads();
        rows_gemm<RB, D, F, 1>(&s.Fh[0][0], a.W + o.w_2, a.W + o.b_2, &s.X[0][0]);
        __syncthreads();
    }
    rows_ln(s.X, s.A, a.W + a.lnf_g, a.W + a.lnf_b);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int r = w; r < RB; r += NT / 32) {
        const float v = warp_sum(s.A[r][lane] * __ldg(a.W + a.head_w + lane) +
                                 s.A[r][lane + 32] * __ldg(a.W + a.head_w + lane + 32));
        if (lane == 0) s.z[r] = v + __ldg(a.W + a.head_b);
    }
    __syncthreads();
}

// e_beta for a row: W_beta . [sin(w_k beta), cos(w_k beta)] + b_beta, w_k = 2^k / 4.
__device__ void beta_embed(const FArgs& a, double beta, float* out) {
    for (int c = threadIdx.x; c < D; c += NT) {
        float acc = __ldg(a.W + a.beta_b + c);
        const int half = a.fb / 2;
        for (int k = 0; k < half; ++k) {
            const double wk = ldexp(1.0, k) / 4.0;
            acc = fmaf((float)sin(wk * beta), __ldg(a.W + a.beta_w + k * D + c), acc);
            acc = fmaf((float)cos(wk * beta), __ldg(a.W + a.beta_w + (half + k) * D + c), acc);
        }
        out[c] = acc;
    }
}

__device__ __forceinline__ double log_sigmoid(double z) { return z >= 0 ? -log1p(exp(-z)) : z - log1p(exp(z)); }

// Build the rows' inputs: x = E[tok_prev] (t > 0) + P_t + e_beta.
template <int RB>
__device__ void rows_input(Smem<RB>& s, const FArgs& a) {
    for (int e = threadIdx.x; e < RB * D; e += NT) {
        const int r = e / D, c = e - r * D;
        float x = 0.f;
        if (s.valid[r]) {
            const int t = s.t[r];
            x = __ldg(a.pos + (size_t)t * D + c) + s.Eb[r][c];
            if (t > 0) x += __ldg(a.W + a.tok_emb + s.tokprev[r] * D + c);
        }
        s.X[r][c] = x;
    }
}

template <class KT>
__global__ void __launch_bounds__(NT) k_former_forward(const FArgs a) {
    constexpr int RB = 32;
    extern __shared__ __align__(16) unsigned char fsm[];
    Smem<RB>& s = *reinterpret_cast<Smem<RB>*>(fsm);
    KVChunk& kv = *reinterpret_cast<KVChunk*>(fsm + ((sizeof(Smem<RB>) + 15) & ~size_t(15)));
    const int tid = threadIdx.x;
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
        beta_embed(a, a.betas[b], &s.Eb[0][0]);
        __syncthreads();
        if (tid < RB) s.lq[tid] = 0.0;
        for (int e = tid + D; e < RB * D; e += NT) (&s.Eb[0][0])[e] = s.Eb[0][e % D];  // same beta for all rows
        for (int t0 = 0; t0 < a.T; t0 += RB) {
            if (tid < RB) {
                const int t = t0 + tid;
                s.t[tid] = t;
                s.slot[tid] = blockIdx.x;
                s.valid[tid] = t < a.T;
                s.tokprev[tid] = (t > 0 && t < a.T) ? a.tokens[(size_t)b * a.T + t - 1] : 0;
            }
            __syncthreads();
            rows_input(s, a);
            __syncthreads();
            rows_forward<RB, KT>(s, a, &kv);
            if (tid < RB && s.valid[tid]) {
                const int t = s.t[tid];
                const float z = s.z[tid];
                if (a.logits) a.logits[(size_t)b * a.T + t] = z;
                if (t >= a.n_prefix) s.lq[tid] += a.tokens[(size_t)b * a.T + t] ? log_sigmoid(z) : log_sigmoid(-z);
            }
            __syncthreads();
        }
        if (tid == 0) {
            double q = 0.0;
            for (int r = 0; r < RB; ++r) q += s.lq[r];
            a.log_q[b] = q;
        }
        __syncthreads();
    }
}

template <int RB, class KT>
__global__ void __launch_bounds__(NT) k_former_sample(const FArgs a) {
    extern __shared__ __align__(16) unsigned char fsm[];
    Smem<RB>& s = *reinterpret_cast<Smem<RB>*>(fsm);
    const int tid = threadIdx.x;
    const int nblk = (a.B + RB - 1) / RB;
    for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        if (tid < RB) {
            const int b = blk * RB + tid;
            s.slot[tid] = blockIdx.x * RB + tid;
            s.valid[tid] = b < a.B;
            s.lq[tid] = 0.0;
            s.tokprev[tid] = 0;
        }
        for (int r = 0; r < RB; ++r) {
            const int b = min(blk * RB + r, a.B - 1);
            beta_embed(a, a.betas[b], &s.Eb[r][0]);
        }
        __syncthreads();
        for (int t = 0; t < a.T; ++t) {
            if (tid < RB) s.t[tid] = t;
            __syncthreads();
            rows_input(s, a);
            __syncthreads();
            rows_forward<RB, KT>(s, a);
            if (tid < RB && s.valid[tid]) {
                const int b = blk * RB + tid;
                const double z = s.z[tid];
                int tok;
                if (t < a.n_prefix) {
                    tok = a.tokens[(size_t)b * a.n_prefix + t] ? 1 : 0;
                } else {
                    const uint64_t x = tapt_dev::draw(a.streams[b], (uint64_t)t + 1ull);
                    const double u = (double)(x >> 11) * 0x1.0p-53;
                    tok = u < 1.0 / (1.0 + exp(-z)) ? 1 : 0;
                    s.lq[tid] += tok ? log_sigmoid(z) : log_sigmoid(-z);
                }
                a.tok_out[(size_t)b * a.T + t] = (uint8_t)tok;
                s.tokprev[tid] = tok;
            }
            __syncthreads();
        }
        if (tid < RB && s.valid[tid]) a.log_q[blk * RB + tid] = s.lq[tid];
        __syncthreads();
    }
}


// =====================================================================================================
// Tensor-core forward (log_prob): the decoder's dense products on tcgen05 (tc.cuh), layer by layer
// over all rows of all sequences.  A row = (sequence b, position t), row = b * T + t.  Per layer:
//   k_tc_qkv  : LN1(X) -> [Q | K | V] = LN1 . W_qkv + b  (M = 128 rows, N = 192, K = 64) -> Q rows,
//               K / V into the cache (slot = sequence)
//   k_tc_attn : causal attention of 32-row blocks of one sequence over its cached keys (CUDA cores,
//               the flash-style rows_attention_fwd) -> O rows
//   k_tc_mlp  : X += O . W_o + b_o;  H = GELU(LN2(X) . W_1 + b_1) (N = 128);  X += H . W_2 + b_2
//               (K = 128): three MMAs per 128-row tile with the epilogues between them
// then k_tc_head: final LayerNorm, head, log q per sequence.  Weights are staged once per persistent
// CTA as bf16 hi / lo splits (bf16x3, ~fp32 accuracy); activations are split per tile; accumulators
// live in TMEM and come back with tcgen05.ld (thread = row).
// =====================================================================================================

struct TcArgs {
    FArgs f;
    int rows, T, B;
    float* X;         // [rows][D] residual stream
    float* Qb;        // [rows][D] queries
    float* O;         // [rows][D] attention outputs
    const float* Eb;  // [B][D] beta embeddings
    // K/V as tensor-core operand tiles for k_tc_attn_mma (null: the fp32 cache for k_tc_attn):
    // [B][L][ceil(T/32)] chunks of 32 keys x [2 heads][K hi | K lo | V^T hi | V^T lo] (2 KB each)
    uint8_t* kvt;
    int nchunk;
};

constexpr int kChunkKeys = 32;                                     // keys per attention chunk
constexpr int kChunkTile = kChunkKeys * 32 * 2;                    // one 32 x 32 bf16 tile (2 KB)
constexpr int kChunkBytes = 2 * 4 * kChunkTile;                    // both heads, K / V, hi / lo: 16 KB

constexpr int kTcThreads = 128;

__global__ void k_tc_beta(const FArgs a, float* Eb) { beta_embed(a, a.betas[blockIdx.x], Eb + (size_t)blockIdx.x * D); }

// x = P_t + e_beta (+ E[tok_{t-1}] for t > 0), as rows_input
__global__ void k_tc_embed(const TcArgs a) {
    const size_t n = (size_t)a.rows * D;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int row = (int)(e / D), c = (int)(e % D);
        const int b = row / a.T, t = row - b * a.T;
        float x = __ldg(a.f.pos + (size_t)t * D + c) + a.Eb[(size_t)b * D + c];
        if (t > 0) x += __ldg(a.f.W + a.f.tok_emb + a.f.tokens[(size_t)b * a.T + t - 1] * D + c);
        a.X[e] = x;
    }
}

// LayerNorm of one row held in registers (eps 1e-5, the rows_ln formula)
__device__ __forceinline__ void row_ln(const float (&x)[D], float (&y)[D], const float* g, const float* bb) {
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) s += x[c];
    const float mu = s * (1.0f / D);
    float v = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) v += (x[c] - mu) * (x[c] - mu);
    const float inv = rsqrtf(v * (1.0f / D) + 1e-5f);
#pragma unroll
    for (int c = 0; c < D; ++c) y[c] = (x[c] - mu) * inv * __ldg(g + c) + __ldg(bb + c);
}

template <int K>
__device__ __forceinline__ void row_to_tile(uint8_t* hi, uint8_t* lo, int r, const float* y) {
#pragma unroll
    for (int k0 = 0; k0 < K; k0 += 8) {
        float x8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x8[i] = y[k0 + i];
        tapt_tc::store_row8(hi, lo, r, k0, K, x8);
    }
}

// W [K][N] row-major (input k, output n) -> B tiles [N][K] K-major, hi / lo
template <int N, int K>
__device__ void stage_weights(uint8_t* hi, uint8_t* lo, const float* W) {
    for (int n = threadIdx.x; n < N; n += blockDim.x)
        for (int k0 = 0; k0 < K; k0 += 8) {
            float x8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x8[i] = __ldg(W + (size_t)(k0 + i) * N + n);
            tapt_tc::store_row8(hi, lo, n, k0, K, x8);
        }
}

__device__ __forceinline__ void tc_sync() {
    tapt_tc::fence_async_smem();
    tapt_tc::fence_before();
    __syncthreads();
    tapt_tc::fence_after();
}

template <int N, int K>
__device__ __forceinline__ void tc_gemm(uint32_t tmem, const uint8_t* ah, const uint8_t* al, const uint8_t* bh,
                                        const uint8_t* bl, uint64_t* bar, uint32_t& phase) {
    if (threadIdx.x == 0) {
        tapt_tc::mma_x3<N, K>(tmem, ah, al, bh, bl);
        tapt_tc::mma_commit(bar);
    }
    tapt_tc::bar_wait(bar, phase);
    phase ^= 1u;
    tapt_tc::fence_after();
}

template <class KT>
__global__ void __launch_bounds__(kTcThreads) k_tc_qkv(const TcArgs a, int l) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* wh = sm;                    // [192][64] bf16
    uint8_t* wl = wh + 3 * D * D * 2;
    uint8_t* ah = wl + 3 * D * D * 2;    // [128][64] bf16
    uint8_t* al = ah + 128 * D * 2;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    const LayerOff& o = a.f.lay[l];
    stage_weights<3 * D, D>(wh, wl, a.f.W + o.w_qkv);
    if (tid == 0) tapt_tc::bar_init(&bar, 1);
    if (warp == 0) tapt_tc::tmem_alloc(&tbase, 256);
    tc_sync();
    const uint32_t tm = tbase, lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t phase = 0;
    const int ntiles = (a.rows + 127) / 128;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row = tile * 128 + tid;
        const bool valid = row < a.rows;
        {
            float x[D], y[D];
#pragma unroll
            for (int c = 0; c < D; c += 4) {
                const float4 v = valid ? *reinterpret_cast<const float4*>(a.X + (size_t)row * D + c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                x[c] = v.x;
                x[c + 1] = v.y;
                x[c + 2] = v.z;
                x[c + 3] = v.w;
            }
            row_ln(x, y, a.f.W + o.ln1_g, a.f.W + o.ln1_b);
            row_to_tile<D>(ah, al, tid, y);
        }
        tc_sync();
        tc_gemm<3 * D, D>(tm, ah, al, wh, wl, &bar, phase);
        {  // tcgen05.ld is warp-collective: every lane loads, valid rows store
            const int b = row / a.T, t = row - b * a.T;
            const size_t kv = ((((size_t)b * a.f.L + l) * a.T + t) * 2) * D;
            const float* bias = a.f.W + o.b_qkv;
#pragma unroll 1
            for (int c = 0; c < 3 * D; c += 16) {
                float v[16];
                tapt_tc::tmem_ld16(tm + lane_base + c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += __ldg(bias + c + i);
                if (valid && c < D) {
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4*>(a.Qb + (size_t)row * D + c + i) =
                            make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                } else if (valid && !a.kvt) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) KVT<KT>::st(a.f.cache, kv + (c - D) + i, v[i]);
                } else if (valid) {  // operand tiles of this key's chunk: K row j; V^T column j
                    const int j = t % kChunkKeys, isv = c >= 2 * D, hh = ((c - D) % D) / DH, d0 = (c - D) % DH;
                    uint8_t* blk = a.kvt + (((size_t)b * a.f.L + l) * a.nchunk + t / kChunkKeys) * kChunkBytes +
                                   (size_t)hh * 4 * kChunkTile;
                    if (!isv) {
#pragma unroll
                        for (int k0 = 0; k0 < 16; k0 += 8) {
                            float x8[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) x8[i] = v[k0 + i];
                            tapt_tc::store_row8(blk, blk + kChunkTile, j, d0 + k0, 32, x8);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            __nv_bfloat16 hi, lo;
                            tapt_tc::split_bf16(v[i], hi, lo);
                            const uint32_t off = tapt_tc::kmajor_off(d0 + i, j, kChunkKeys);
                            *reinterpret_cast<__nv_bfloat16*>(blk + 2 * kChunkTile + off) = hi;
                            *reinterpret_cast<__nv_bfloat16*>(blk + 3 * kChunkTile + off) = lo;
                        }
                    }
                }
            }
        }
        tapt_tc::fence_before();
        __syncthreads();
    }
    if (warp == 0) tapt_tc::tmem_free(tm, 256);
}

template <class KT>
__global__ void __launch_bounds__(NT) k_tc_attn(const TcArgs a, int l) {
    extern __shared__ __align__(16) unsigned char fsm[];
    Smem<32>& s = *reinterpret_cast<Smem<32>*>(fsm);
    KVChunk& kv = *reinterpret_cast<KVChunk*>(fsm + ((sizeof(Smem<32>) + 15) & ~size_t(15)));
    const int b = blockIdx.y, t0 = blockIdx.x * 32;
    if (threadIdx.x < 32) {
        const int t = t0 + threadIdx.x;
        s.t[threadIdx.x] = t;
        s.slot[threadIdx.x] = b;
        s.valid[threadIdx.x] = t < a.T;
    }
    for (int e = threadIdx.x; e < 32 * D; e += NT) {
        const int r = e / D, c = e - r * D;
        s.Q[r][c] = t0 + r < a.T ? a.Qb[((size_t)b * a.T + t0 + r) * D + c] : 0.f;
    }
    __syncthreads();
    rows_attention_fwd<32, KT>(s, kv, a.f, l);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * D; e += NT) {
        const int r = e / D, c = e - r * D;
        if (t0 + r < a.T) a.O[((size_t)b * a.T + t0 + r) * D + c] = s.O[r][c];
    }
}

__global__ void __launch_bounds__(kTcThreads) k_tc_mlp(const TcArgs a, int l) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* woh = sm;                       // [64][64]
    uint8_t* wol = woh + D * D * 2;
    uint8_t* w1h = wol + D * D * 2;          // [128][64]
    uint8_t* w1l = w1h + F * D * 2;
    uint8_t* w2h = w1l + F * D * 2;          // [64][128]
    uint8_t* w2l = w2h + D * F * 2;
    uint8_t* t1h = w2l + D * F * 2;          // [128][64] activations (O, then LN2)
    uint8_t* t1l = t1h + 128 * D * 2;
    uint8_t* t2h = t1l + 128 * D * 2;        // [128][128] hidden
    uint8_t* t2l = t2h + 128 * F * 2;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    const LayerOff& o = a.f.lay[l];
    stage_weights<D, D>(woh, wol, a.f.W + o.w_o);
    stage_weights<F, D>(w1h, w1l, a.f.W + o.w_1);
    stage_weights<D, F>(w2h, w2l, a.f.W + o.w_2);
    if (tid == 0) tapt_tc::bar_init(&bar, 1);
    if (warp == 0) tapt_tc::tmem_alloc(&tbase, 256);
    tc_sync();
    const uint32_t tm = tbase, lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t c_o = 0, c_1 = 64, c_2 = 192;  // TMEM columns of the three products
    uint32_t phase = 0;
    const int ntiles = (a.rows + 127) / 128;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row = tile * 128 + tid;
        const bool valid = row < a.rows;
        float x[D];
        {
            float y[D];
#pragma unroll
            for (int c = 0; c < D; c += 4) {
                const float4 v = valid ? *reinterpret_cast<const float4*>(a.O + (size_t)row * D + c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                y[c] = v.x;
                y[c + 1] = v.y;
                y[c + 2] = v.z;
                y[c + 3] = v.w;
            }
            row_to_tile<D>(t1h, t1l, tid, y);
#pragma unroll
            for (int c = 0; c < D; c += 4) {
                const float4 v = valid ? *reinterpret_cast<const float4*>(a.X + (size_t)row * D + c)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                x[c] = v.x;
                x[c + 1] = v.y;
                x[c + 2] = v.z;
                x[c + 3] = v.w;
            }
        }
        tc_sync();
        tc_gemm<D, D>(tm + c_o, t1h, t1l, woh, wol, &bar, phase);
        {  // X += O W_o + b_o, then LN2 into the activation tile
#pragma unroll
            for (int c = 0; c < D; c += 16) {
                float v[16];
                tapt_tc::tmem_ld16(tm + lane_base + c_o + c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) x[c + i] += v[i] + __ldg(a.f.W + o.b_o + c + i);
            }
            float y[D];
            row_ln(x, y, a.f.W + o.ln2_g, a.f.W + o.ln2_b);
            row_to_tile<D>(t1h, t1l, tid, y);
        }
        tc_sync();
        tc_gemm<F, D>(tm + c_1, t1h, t1l, w1h, w1l, &bar, phase);
#pragma unroll 1
        for (int c = 0; c < F; c += 16) {  // H = GELU(LN2 W_1 + b_1) into the hidden tile
            float v[16];
            tapt_tc::tmem_ld16(tm + lane_base + c_1 + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = gelu(v[i] + __ldg(a.f.W + o.b_1 + c + i));
#pragma unroll
            for (int h = 0; h < 16; h += 8) {
                float x8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) x8[i] = v[h + i];
                tapt_tc::store_row8(t2h, t2l, tid, c + h, F, x8);
            }
        }
        tc_sync();
        tc_gemm<D, F>(tm + c_2, t2h, t2l, w2h, w2l, &bar, phase);
#pragma unroll
        for (int c = 0; c < D; c += 16) {  // X += H W_2 + b_2
            float v[16];
            tapt_tc::tmem_ld16(tm + lane_base + c_2 + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) x[c + i] += v[i] + __ldg(a.f.W + o.b_2 + c + i);
        }
        if (valid)
#pragma unroll
            for (int c = 0; c < D; c += 4)
                *reinterpret_cast<float4*>(a.X + (size_t)row * D + c) = make_float4(x[c], x[c + 1], x[c + 2], x[c + 3]);
        tapt_tc::fence_before();
        __syncthreads();
    }
    if (warp == 0) tapt_tc::tmem_free(tm, 256);
}

// Causal attention of one 128-position query block of one sequence on the tensor cores (flash
// style).  256 threads: warpgroup h (warps 4h .. 4h+3) owns head h, thread = query row (TMEM lane).
// K and V arrive as ready-made operand tiles (k_tc_qkv writes them: per 32-key chunk, K [key][dim]
// and V^T [dim][key], bf16 hi / lo, both heads, 16 KB), copied into shared memory by cp.async.bulk
// into a ring of 3 buffers, two chunks ahead.  Software-pipelined so each chunk costs ONE MMA round
// trip: after the softmax of chunk c (scores from TMEM, causal mask, online max / sum, P as a hi / lo
// tile) one thread issues P_c V_c and S_{c+1} = Q K_{c+1}^T for both heads under a single commit; the
// next iteration folds P_c V_c into the row's fp32 accumulator and starts the softmax of c + 1.
// grid (ceil(T / 128), B).
constexpr int kAttnThreads = 256, kKvBufs = 3;

__global__ void __launch_bounds__(kAttnThreads) k_tc_attn_mma(const TcArgs a, int l) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int QT = 128 * DH * 2, PT = 128 * kChunkKeys * 2;
    uint8_t* qh = sm;                          // [2 heads][128][32] hi
    uint8_t* ql = qh + 2 * QT;                 //                    lo
    uint8_t* kv = ql + 2 * QT;                 // [3 buffers][16 KB chunk]
    uint8_t* ph = kv + kKvBufs * kChunkBytes;  // [2 heads][128][32 keys]
    uint8_t* pl = ph + 2 * PT;
    __shared__ uint64_t bar, kvbar[kKvBufs];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, h = tid >> 7, r = tid & 127;
    const int b = blockIdx.y, q0 = blockIdx.x * 128, t = q0 + r;
    const int tq = min(t, a.T - 1);  // rows past the sequence end attend like its last row (not stored)
    const int kmax = min(q0 + 127, a.T - 1), nch = kmax / kChunkKeys + 1;
    const uint8_t* src = a.kvt + (((size_t)b * a.f.L + l) * a.nchunk) * kChunkBytes;
    auto fetch = [&](int ci) {  // thread 0
        uint64_t* kb = &kvbar[ci % kKvBufs];
        tapt_dev::mbar_expect_tx(kb, kChunkBytes);
        tapt_dev::bulk_g2s(kv + (ci % kKvBufs) * kChunkBytes, src + (size_t)ci * kChunkBytes, kChunkBytes, kb);
    };
    auto issue_qk = [&](int ci) {  // thread 0: S_h = Q_h K_h^T of chunk ci, both heads
        const uint8_t* kb = kv + (ci % kKvBufs) * kChunkBytes;
        tapt_tc::bar_wait(&kvbar[ci % kKvBufs], (uint32_t)(ci / kKvBufs) & 1u);
        tapt_tc::fence_after();
        tapt_tc::mma_x3<kChunkKeys, DH>(tbase + 0, qh, ql, kb, kb + kChunkTile);
        tapt_tc::mma_x3<kChunkKeys, DH>(tbase + kChunkKeys, qh + QT, ql + QT, kb + 4 * kChunkTile, kb + 5 * kChunkTile);
    };
    if (tid == 0) {
        tapt_tc::bar_init(&bar, 1);
        for (int i = 0; i < kKvBufs; ++i) tapt_tc::bar_init(&kvbar[i], 1);
        fetch(0);
        if (nch > 1) fetch(1);
    }
    {  // Q of this row, this head
        const float* q = a.Qb + ((size_t)b * a.T + tq) * D + h * DH;
#pragma unroll
        for (int k0 = 0; k0 < DH; k0 += 8) {
            float x8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x8[i] = q[k0 + i];
            tapt_tc::store_row8(qh + h * QT, ql + h * QT, r, k0, DH, x8);
        }
    }
    if (warp == 0) tapt_tc::tmem_alloc(&tbase, 256);
    tc_sync();
    const uint32_t tm = tbase, lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t cS = (uint32_t)kChunkKeys * h, cO = 128u + 32u * h;  // TMEM: scores [0, 64), P V [128, 192)
    const float scale = rsqrtf((float)DH);
    float m = -INFINITY, lsum = 0.f, corr = 1.f, o[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) o[d] = 0.f;
    uint32_t phase = 0;
    if (tid == 0) {
        issue_qk(0);
        tapt_tc::mma_commit(&bar);
    }
    for (int ci = 0; ci <= nch; ++ci) {
        tapt_tc::bar_wait(&bar, phase);  // S_ci and P_{ci-1} V_{ci-1} have landed
        phase ^= 1u;
        tapt_tc::fence_after();
        if (ci > 0) {  // fold P V of the previous chunk in, with that chunk's rescale
#pragma unroll
            for (int c = 0; c < DH; c += 16) {
                float w16[16];
                tapt_tc::tmem_ld16(tm + lane_base + cO + c, w16);
#pragma unroll
                for (int i = 0; i < 16; ++i) o[c + i] = o[c + i] * corr + w16[i];
            }
        }
        if (ci == nch) break;
        if (tid == 0 && ci + 2 < nch) fetch(ci + 2);  // its buffer held chunk ci - 1, whose MMAs have retired
        const int c0 = ci * kChunkKeys;
        float v[kChunkKeys];
#pragma unroll
        for (int c = 0; c < kChunkKeys; c += 16) {
            float w16[16];
            tapt_tc::tmem_ld16(tm + lane_base + cS + c, w16);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[c + i] = c0 + c + i <= tq ? w16[i] * scale : -INFINITY;
        }
        float mx = m;
#pragma unroll
        for (int i = 0; i < kChunkKeys; ++i) mx = fmaxf(mx, v[i]);
        corr = __expf(m - mx);
        float ps = 0.f;
#pragma unroll
        for (int i = 0; i < kChunkKeys; ++i) {
            v[i] = c0 + i <= tq ? __expf(v[i] - mx) : 0.f;
            ps += v[i];
        }
#pragma unroll
        for (int k0 = 0; k0 < kChunkKeys; k0 += 8) {
            float x8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x8[i] = v[k0 + i];
            tapt_tc::store_row8(ph + h * PT, pl + h * PT, r, k0, kChunkKeys, x8);
        }
        lsum = lsum * corr + ps;
        m = mx;
        tc_sync();  // P written; the scores and the P V columns have been read
        if (tid == 0) {
            const uint8_t* kb = kv + (ci % kKvBufs) * kChunkBytes;
            tapt_tc::mma_x3<DH, kChunkKeys>(tm + 128, ph, pl, kb + 2 * kChunkTile, kb + 3 * kChunkTile);
            tapt_tc::mma_x3<DH, kChunkKeys>(tm + 128 + DH, ph + PT, pl + PT, kb + 6 * kChunkTile, kb + 7 * kChunkTile);
            if (ci + 1 < nch) issue_qk(ci + 1);
            tapt_tc::mma_commit(&bar);
        }
    }
    if (t < a.T) {
        float* dst = a.O + ((size_t)b * a.T + t) * D + h * DH;
        const float inv = 1.f / lsum;
#pragma unroll
        for (int d = 0; d < DH; d += 4)
            *reinterpret_cast<float4*>(dst + d) = make_float4(o[d] * inv, o[d + 1] * inv, o[d + 2] * inv, o[d + 3] * inv);
    }
    tapt_tc::fence_before();
    __syncthreads();
    if (warp == 0) tapt_tc::tmem_free(tm, 256);
}

// Final LayerNorm + head per row, log q per sequence (positions >= n_prefix).  grid B, NT threads.
__global__ void __launch_bounds__(NT) k_tc_head(const TcArgs a) {
    __shared__ double part[NT];
    const int b = blockIdx.x;
    double lq = 0.0;
    for (int t = threadIdx.x; t < a.T; t += NT) {
        const size_t row = (size_t)b * a.T + t;
        float x[D], y[D];
#pragma unroll
        for (int c = 0; c < D; c += 4) {
            const float4 v = *reinterpret_cast<const float4*>(a.X + row * D + c);
            x[c] = v.x;
            x[c + 1] = v.y;
            x[c + 2] = v.z;
            x[c + 3] = v.w;
        }
        row_ln(x, y, a.f.W + a.f.lnf_g, a.f.W + a.f.lnf_b);
        float z = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) z = fmaf(y[c], __ldg(a.f.W + a.f.head_w + c), z);
        z += __ldg(a.f.W + a.f.head_b);
        if (a.f.logits) a.f.logits[row] = z;
        if (t >= a.f.n_prefix) lq += a.f.tokens[row] ? log_sigmoid(z) : log_sigmoid(-z);
    }
    part[threadIdx.x] = lq;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.f.log_q[b] = part[0];
}

}  // namespace tapt_former_dev

using namespace tapt_former_dev;

// ==================================================================== host ===

namespace {

#define FCUDA(expr)                                                                                      \
    do {                                                                                                 \
        cudaError_t e_ = (expr);                                                                         \
        if (e_ != cudaSuccess) throw tapt::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class Fn>
tapt_status fguard(Fn&& f) {
    try {
        f();
        return TAPT_OK;
    } catch (const tapt::ConfigError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_CONFIG;
    } catch (const tapt::DimensionError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_DIMENSION;
    } catch (const tapt::SizeError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_SIZE;
    } catch (const tapt::FormatError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_FORMAT;
    } catch (const tapt::NumericError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_NUMERIC;
    } catch (const tapt::CudaError& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_CUDA;
    } catch (const std::exception& e) {
        tapt_host::set_last_error(e.what());
        return TAPT_ERR_INTERNAL;
    }
}

struct Layout {
    size_t total = 0;
    int tok_emb, beta_w, beta_b, lnf_g, lnf_b, head_w, head_b;
    std::vector<LayerOff> lay;
    // (offset, size, fan_in; fan_in 0 = bias/zero, -1 = LN gain/one) for initialisation
    struct Item {
        size_t off, size;
        int fan_in;
    };
    std::vector<Item> items;
};

void check_config(const tapt_former_config* c) {
    if (!c) throw tapt::ConfigError("null former config");
    if (c->d_model == 0 || c->heads == 0 || c->ffn == 0 || c->layers == 0 || c->max_len == 0)
        throw tapt::ConfigError("former dimensions must be >= 1");
    if (c->d_model % c->heads) throw tapt::ConfigError("d_model must be divisible by heads");
    if (c->beta_features == 0 || c->beta_features % 2) throw tapt::ConfigError("beta_features must be even and >= 2");
}

Layout make_layout(const tapt_former_config& c) {
    Layout L;
    const int d = (int)c.d_model, f = (int)c.ffn, fb = (int)c.beta_features;
    size_t o = 0;
    auto put = [&](size_t n, int fan) {
        const size_t at = o;
        L.items.push_back({at, n, fan});
        o += n;
        return (int)at;
    };
    L.tok_emb = put(2 * (size_t)d, 1);
    L.beta_w = put((size_t)fb * d, fb);
    L.beta_b = put(d, 0);
    for (uint32_t l = 0; l < c.layers; ++l) {
        LayerOff y;
        y.ln1_g = put(d, -1);
        y.ln1_b = put(d, 0);
        y.w_qkv = put((size_t)d * 3 * d, d);
        y.b_qkv = put(3 * (size_t)d, 0);
        y.w_o = put((size_t)d * d, d);
        y.b_o = put(d, 0);
        y.ln2_g = put(d, -1);
        y.ln2_b = put(d, 0);
        y.w_1 = put((size_t)d * f, d);
        y.b_1 = put(f, 0);
        y.w_2 = put((size_t)f * d, f);
        y.b_2 = put(d, 0);
        L.lay.push_back(y);
    }
    L.lnf_g = put(d, -1);
    L.lnf_b = put(d, 0);
    L.head_w = put(d, d);
    L.head_b = put(1, 0);
    L.total = o;
    return L;
}

}  // namespace

struct tapt_former_s {
    tapt_former_config cfg{};
    Layout lay;
    std::vector<float> params;
    float* dW = nullptr;
    float* dpos = nullptr;
    void* cache = nullptr;
    size_t cache_n = 0;  // bytes
    int kv16 = 0;        // K/V cache in bf16 (tapt_former_set_kv_bf16)
    int tc = 1;          // log_prob's dense products on the tensor cores (tapt_former_set_tensor_cores)
    float* tcbuf = nullptr;  // X | Q | O | e_beta of the tensor-core forward
    size_t tcbuf_n = 0;
    void* tmp = nullptr;
    size_t tmp_n = 0;
    ~tapt_former_s() {
        if (dW) cudaFree(dW);
        if (dpos) cudaFree(dpos);
        if (cache) cudaFree(cache);
        if (tmp) cudaFree(tmp);
        if (tcbuf) cudaFree(tcbuf);
    }
    float* need_tcbuf(size_t floats) {
        if (floats > tcbuf_n) {
            if (tcbuf) cudaFree(tcbuf);
            tcbuf = nullptr;
            FCUDA(cudaMalloc(&tcbuf, floats * sizeof(float)));
            tcbuf_n = floats;
        }
        return tcbuf;
    }
    void upload() {
        if (dW) return;
        FCUDA(cudaMalloc(&dW, params.size() * sizeof(float)));
        FCUDA(cudaMemcpy(dW, params.data(), params.size() * sizeof(float), cudaMemcpyHostToDevice));
        const int d = (int)cfg.d_model;
        std::vector<float> P((size_t)cfg.max_len * d);
        for (uint32_t t = 0; t < cfg.max_len; ++t)
            for (int i = 0; i < d / 2; ++i) {
                const double ang = (double)t / std::pow(10000.0, 2.0 * i / d);
                P[(size_t)t * d + 2 * i] = (float)std::sin(ang);
                P[(size_t)t * d + 2 * i + 1] = (float)std::cos(ang);
            }
        FCUDA(cudaMalloc(&dpos, P.size() * sizeof(float)));
        FCUDA(cudaMemcpy(dpos, P.data(), P.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    void* need_cache(size_t n) {  // n elements of the configured K/V type
        const size_t bytes = n * (kv16 ? 2 : 4);
        if (bytes > cache_n) {
            if (cache) cudaFree(cache);
            cache = nullptr;
            FCUDA(cudaMalloc(&cache, bytes));
            cache_n = bytes;
        }
        return cache;
    }
    uint8_t* need_tmp(size_t bytes) {
        if (bytes > tmp_n) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            FCUDA(cudaMalloc(&tmp, bytes));
            tmp_n = bytes;
        }
        return static_cast<uint8_t*>(tmp);
    }
    FArgs args() const {
        FArgs a{};
        a.W = dW;
        a.tok_emb = lay.tok_emb;
        a.beta_w = lay.beta_w;
        a.beta_b = lay.beta_b;
        a.lnf_g = lay.lnf_g;
        a.lnf_b = lay.lnf_b;
        a.head_w = lay.head_w;
        a.head_b = lay.head_b;
        for (size_t l = 0; l < lay.lay.size(); ++l) a.lay[l] = lay.lay[l];
        a.L = (int)cfg.layers;
        a.fb = (int)cfg.beta_features;
        a.pos = dpos;
        return a;
    }
};

namespace {

void check_device_shape(const tapt_former_config& c) {
    if (c.d_model != (uint32_t)D || c.d_model / c.heads != (uint32_t)DH || c.ffn != (uint32_t)F)
        throw tapt::SizeError("device kernels support d_model = 64, 32-wide heads, ffn = 128 (the SPEC default)");
    if (c.layers > (uint32_t)kMaxL) throw tapt::SizeError("at most 16 layers");
}

int sm_count() {
    int dev = 0, n = 0;
    FCUDA(cudaGetDevice(&dev));
    FCUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

tapt_former_s* check_former(tapt_former_t f) {
    if (!f) throw tapt::ConfigError("null former handle");
    return f;
}

tapt_former_s* create_former(const tapt_former_config* c, const float* params) {
    check_config(c);
    if (!params) throw tapt::ConfigError("null parameters");
    auto f = std::make_unique<tapt_former_s>();
    f->cfg = *c;
    f->lay = make_layout(*c);
    f->params.assign(params, params + f->lay.total);
    for (float v : f->params)
        if (!std::isfinite(v)) throw tapt::NumericError("non-finite parameter");
    check_device_shape(*c);
    return f.release();  // device copies are made on first use (create/save/load work without a GPU)
}

// log_prob on the tensor cores (k_tc_*): sequences in chunks that keep the K/V cache and the row
// buffers under ~8 GB; per chunk embed, then per layer QKV (tcgen05) -> attention (CUDA cores) ->
// out-projection + FFN (tcgen05), then head and log q.
template <class KT>
void log_prob_tc(tapt_former_s* f, const FArgs& a0) {
    const int T = a0.T, L = (int)f->cfg.layers, nsm = sm_count();
    const int nchunk = (T + kChunkKeys - 1) / kChunkKeys;
    // attention products on the tensor cores too (fp32 cache only); TAPT_FORMER_ATTN_TC=0: CUDA cores
    const char* ae = std::getenv("TAPT_FORMER_ATTN_TC");
    const bool attn_tc = sizeof(KT) == 4 && !(ae && std::atoi(ae) == 0);
    const size_t per_seq = (size_t)3 * T * D * 4 + D * 4 +
                           (attn_tc ? (size_t)L * nchunk * kChunkBytes : (size_t)L * T * 2 * D * sizeof(KT));
    const int Bc = (int)std::max<size_t>(1, std::min<size_t>((size_t)a0.B, (size_t)(16ull << 30) / per_seq));
    const size_t smem_qkv = (size_t)2 * 3 * D * D * 2 + (size_t)2 * 128 * D * 2;
    const size_t smem_mlp = (size_t)2 * (D * D + F * D + D * F) * 2 + (size_t)2 * 128 * D * 2 + (size_t)2 * 128 * F * 2;
    const size_t smem_attn = ((sizeof(Smem<32>) + 15) & ~size_t(15)) + sizeof(KVChunk);
    FCUDA(cudaFuncSetAttribute(k_tc_qkv<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_qkv));
    FCUDA(cudaFuncSetAttribute(k_tc_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mlp));
    FCUDA(cudaFuncSetAttribute(k_tc_attn<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_attn));
    const size_t smem_amma =
        (size_t)2 * (2 * 128 * DH * 2) + (size_t)kKvBufs * kChunkBytes + (size_t)2 * (2 * 128 * kChunkKeys * 2);
    FCUDA(cudaFuncSetAttribute(k_tc_attn_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_amma));
    for (int b0 = 0; b0 < a0.B; b0 += Bc) {
        const int nb = std::min(Bc, a0.B - b0);
        TcArgs t{};
        t.f = a0;
        t.f.tokens = a0.tokens + (size_t)b0 * T;
        t.f.betas = a0.betas + b0;
        t.f.log_q = a0.log_q + b0;
        t.f.logits = a0.logits ? a0.logits + (size_t)b0 * T : nullptr;
        t.f.B = nb;
        t.f.cache = attn_tc ? nullptr : f->need_cache((size_t)nb * L * T * 2 * D);
        t.rows = nb * T;
        t.T = T;
        t.B = nb;
        const size_t kvt_floats = attn_tc ? ((size_t)nb * L * nchunk * kChunkBytes + 3) / 4 : 0;
        float* buf = f->need_tcbuf((size_t)3 * t.rows * D + (size_t)nb * D + kvt_floats);
        t.X = buf;
        t.Qb = buf + (size_t)t.rows * D;
        t.O = buf + (size_t)2 * t.rows * D;
        t.Eb = buf + (size_t)3 * t.rows * D;
        t.nchunk = nchunk;
        t.kvt = nullptr;
        if (attn_tc) {  // chunk tiles; keys past T stay zero (finite operands for the masked products)
            t.kvt = reinterpret_cast<uint8_t*>(buf + (size_t)3 * t.rows * D + (size_t)nb * D);
            if (T % kChunkKeys)  // only the last chunk of each (sequence, layer) has keys past T
                FCUDA(cudaMemset2DAsync(t.kvt + (size_t)(nchunk - 1) * kChunkBytes, (size_t)nchunk * kChunkBytes, 0,
                                        kChunkBytes, (size_t)nb * L));
        }
        const int ntiles = (t.rows + 127) / 128;
        k_tc_beta<<<nb, D>>>(t.f, const_cast<float*>(t.Eb));
        k_tc_embed<<<std::min(nsm * 8, (t.rows * D + 255) / 256), 256>>>(t);
        for (int l = 0; l < L; ++l) {
            k_tc_qkv<KT><<<std::min(ntiles, 2 * nsm), kTcThreads, smem_qkv>>>(t, l);
            if (attn_tc)
                k_tc_attn_mma<<<dim3((T + 127) / 128, nb), kAttnThreads, smem_amma>>>(t, l);
            else
                k_tc_attn<KT><<<dim3((T + 31) / 32, nb), NT, smem_attn>>>(t, l);
            k_tc_mlp<<<std::min(ntiles, nsm), kTcThreads, smem_mlp>>>(t, l);
        }
        k_tc_head<<<nb, NT>>>(t);
        tapt_host::note_launches(3 + 3 * L);
        FCUDA(cudaGetLastError());
    }
}

template <int RB, class K>
void launch_rows(K kernel, int grid, const FArgs& a, size_t extra = 0) {
    const int smem = (int)(((sizeof(Smem<RB>) + 15) & ~size_t(15)) + extra);
    FCUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kernel<<<grid, NT, smem>>>(a);
    tapt_host::note_launches(1);
    FCUDA(cudaGetLastError());
}

}  // namespace

extern "C" {

size_t tapt_former_param_count(const tapt_former_config* c) {
    if (!c || c->d_model == 0 || c->beta_features == 0) return 0;
    return make_layout(*c).total;
}

tapt_status tapt_former_init_params(const tapt_former_config* c, uint64_t seed, double scale, float* params) {
    return fguard([&] {
        check_config(c);
        if (!params) throw tapt::ConfigError("null parameter buffer");
        const Layout L = make_layout(*c);
        tapt::RngStream r = tapt::RngStream::derive(seed, {0x77});
        for (const auto& it : L.items) {
            for (size_t k = 0; k < it.size; ++k) {
                float v;
                if (it.fan_in == 0) {
                    v = 0.f;
                } else if (it.fan_in < 0) {
                    v = 1.f;
                } else {  // Box-Muller on two 53-bit uniforms
                    const double u1 = 1.0 - r.uniform(), u2 = r.uniform();
                    const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
                    v = (float)(scale * g / std::sqrt((double)it.fan_in));
                }
                params[it.off + k] = v;
            }
        }
    });
}

tapt_status tapt_former_create(const tapt_former_config* c, const float* params, tapt_former_t* out) {
    return fguard([&] {
        if (!out) throw tapt::ConfigError("null output handle");
        *out = create_former(c, params);
    });
}

tapt_status tapt_former_destroy(tapt_former_t f) {
    delete f;
    return TAPT_OK;
}

tapt_status tapt_former_get(tapt_former_t f, tapt_former_config* c, float* params) {
    return fguard([&] {
        check_former(f);
        if (c) *c = f->cfg;
        if (params) std::memcpy(params, f->params.data(), f->params.size() * sizeof(float));
    });
}

tapt_status tapt_former_save(tapt_former_t f, const char* path) {
    return fguard([&] {
        check_former(f);
        if (!path) throw tapt::ConfigError("null path");
        std::ofstream o(path, std::ios::binary);
        if (!o) throw tapt::FormatError(std::string("cannot open ") + path);
        o.write("ISFW1", 5);
        const uint32_t hdr[8] = {1u, f->cfg.d_model, f->cfg.heads, f->cfg.ffn, f->cfg.layers, f->cfg.max_len,
                                 f->cfg.beta_features, (uint32_t)f->params.size()};
        o.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));  // little-endian hosts only (x86-64, aarch64)
        o.write(reinterpret_cast<const char*>(f->params.data()), (std::streamsize)(f->params.size() * sizeof(float)));
        if (!o) throw tapt::FormatError("write failed");
    });
}

tapt_status tapt_former_load(const char* path, tapt_former_t* out) {
    return fguard([&] {
        if (!path || !out) throw tapt::ConfigError("null path / output");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw tapt::FormatError(std::string("cannot open ") + path);
        char magic[5];
        in.read(magic, 5);
        if (!in || std::memcmp(magic, "ISFW1", 5) != 0) throw tapt::FormatError("bad ISFW1 magic");
        uint32_t hdr[8];
        in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
        if (!in) throw tapt::FormatError("truncated ISFW1 header");
        if (hdr[0] != 1u) throw tapt::FormatError("unsupported ISFW1 version");
        tapt_former_config c{hdr[1], hdr[2], hdr[3], hdr[4], hdr[5], hdr[6]};
        check_config(&c);
        const size_t n = make_layout(c).total;
        if (hdr[7] != n) throw tapt::FormatError("ISFW1 parameter count does not match its config");
        std::vector<float> p(n);
        in.read(reinterpret_cast<char*>(p.data()), (std::streamsize)(n * sizeof(float)));
        if (!in) throw tapt::FormatError("truncated ISFW1 parameters");
        *out = create_former(&c, p.data());
    });
}

tapt_status tapt_former_set_tensor_cores(tapt_former_t f, int on) {
    return fguard([&] {
        check_former(f);
        f->tc = on ? 1 : 0;
    });
}

tapt_status tapt_former_set_kv_bf16(tapt_former_t f, int bf16) {
    return fguard([&] {
        check_former(f);
        f->kv16 = bf16 ? 1 : 0;
    });
}

tapt_status tapt_former_log_prob(tapt_former_t f, const uint8_t* tokens, uint32_t B, uint32_t T, const double* betas,
                                 uint32_t n_prefix, double* log_q, float* logits) {
    return fguard([&] {
        check_former(f);
        if (!tokens || !betas || !log_q) throw tapt::ConfigError("null tokens / betas / log_q");
        if (T == 0 || T > f->cfg.max_len) throw tapt::SizeError("sequence length must be in [1, max_len]");
        if (n_prefix > T) throw tapt::DimensionError("prefix longer than the sequence");
        if (B == 0) return;
        const int grid = (int)std::min<uint32_t>(B, (uint32_t)sm_count() * 4);
        f->upload();
        FArgs a = f->args();
        a.T = (int)T;
        a.n_prefix = (int)n_prefix;
        a.B = (int)B;
        const size_t tb = (size_t)B * T, off_b = (tb + 255) & ~size_t(255), off_q = off_b + (size_t)B * 8,
                     off_z = off_q + (size_t)B * 8;
        uint8_t* tmp = f->need_tmp(off_z + (logits ? tb * 4 : 0));
        FCUDA(cudaMemcpy(tmp, tokens, tb, cudaMemcpyHostToDevice));
        FCUDA(cudaMemcpy(tmp + off_b, betas, (size_t)B * 8, cudaMemcpyHostToDevice));
        a.tokens = tmp;
        a.betas = reinterpret_cast<const double*>(tmp + off_b);
        a.log_q = reinterpret_cast<double*>(tmp + off_q);
        a.logits = logits ? reinterpret_cast<float*>(tmp + off_z) : nullptr;
        const char* env = std::getenv("TAPT_FORMER_TC");
        // tcgen05 dense products (k_tc_*) with the fp32 K/V cache.  A bf16 cache rounds K and V, so
        // sample / log_prob consistency (the MH correction) needs bit-identical QKV arithmetic in both:
        // with kv16 log_prob keeps the CUDA-core engine the sampler uses.
        const bool tc = f->tc && !f->kv16 && !(env && std::atoi(env) == 0);
        if (!tc) a.cache = f->need_cache((size_t)grid * f->cfg.layers * T * 2 * D);
        if (tc) {
            log_prob_tc<float>(f, a);
        } else if (f->kv16) {
            launch_rows<32>(k_former_forward<__nv_bfloat16>, grid, a, sizeof(KVChunk));
        } else {
            launch_rows<32>(k_former_forward<float>, grid, a, sizeof(KVChunk));
        }
        FCUDA(cudaMemcpy(log_q, a.log_q, (size_t)B * 8, cudaMemcpyDeviceToHost));
        if (logits) FCUDA(cudaMemcpy(logits, a.logits, tb * 4, cudaMemcpyDeviceToHost));
    });
}

tapt_status tapt_former_sample(tapt_former_t f, uint32_t B, uint32_t T, const double* betas, const uint8_t* prefix,
                               uint32_t n_prefix, const uint64_t* streams, uint8_t* tokens, double* log_q) {
    return fguard([&] {
        check_former(f);
        if (!betas || !streams || !tokens || !log_q) throw tapt::ConfigError("null betas / streams / outputs");
        if (T == 0 || T > f->cfg.max_len) throw tapt::SizeError("sequence length must be in [1, max_len]");
        if (n_prefix > T) throw tapt::DimensionError("prefix longer than the sequence");
        if (n_prefix && !prefix) throw tapt::ConfigError("null prefix");
        if (B == 0) return;
        // rows (sequences) per CTA: the largest of 32 / 8 / 4 that still gives two CTAs per SM
        const int nsm = sm_count();
        int RBs = (B + 31) / 32 >= 2u * nsm ? 32 : ((B + 7) / 8 >= 2u * nsm ? 8 : 4);
        if (const char* e = std::getenv("TAPT_FORMER_RB")) RBs = std::atoi(e) >= 32 ? 32 : (std::atoi(e) >= 8 ? 8 : 4);
        const int nblk = (int)((B + RBs - 1) / RBs);
        const int grid = std::min(nblk, nsm * (RBs == 32 ? 4 : 8));
        f->upload();
        FArgs a = f->args();
        a.T = (int)T;
        a.n_prefix = (int)n_prefix;
        a.B = (int)B;
        a.cache = f->need_cache((size_t)grid * RBs * f->cfg.layers * T * 2 * D);
        const size_t pb = (size_t)B * n_prefix, off_b = (pb + 255) & ~size_t(255), off_s = off_b + (size_t)B * 8,
                     off_q = off_s + (size_t)B * 8, off_t = off_q + (size_t)B * 8;
        uint8_t* tmp = f->need_tmp(off_t + (size_t)B * T);
        if (pb) FCUDA(cudaMemcpy(tmp, prefix, pb, cudaMemcpyHostToDevice));
        FCUDA(cudaMemcpy(tmp + off_b, betas, (size_t)B * 8, cudaMemcpyHostToDevice));
        FCUDA(cudaMemcpy(tmp + off_s, streams, (size_t)B * 8, cudaMemcpyHostToDevice));
        a.tokens = tmp;
        a.betas = reinterpret_cast<const double*>(tmp + off_b);
        a.streams = reinterpret_cast<const uint64_t*>(tmp + off_s);
        a.log_q = reinterpret_cast<double*>(tmp + off_q);
        a.tok_out = tmp + off_t;
        if (f->kv16) {
            if (RBs == 32)
                launch_rows<32>(k_former_sample<32, __nv_bfloat16>, grid, a);
            else if (RBs == 8)
                launch_rows<8>(k_former_sample<8, __nv_bfloat16>, grid, a);
            else
                launch_rows<4>(k_former_sample<4, __nv_bfloat16>, grid, a);
        } else {
            if (RBs == 32)
                launch_rows<32>(k_former_sample<32, float>, grid, a);
            else if (RBs == 8)
                launch_rows<8>(k_former_sample<8, float>, grid, a);
            else
                launch_rows<4>(k_former_sample<4, float>, grid, a);
        }
        FCUDA(cudaMemcpy(tokens, a.tok_out, (size_t)B * T, cudaMemcpyDeviceToHost));
        FCUDA(cudaMemcpy(log_q, a.log_q, (size_t)B * 8, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
