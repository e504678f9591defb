// Redundancy-bypassing dispatch (RBD) with one GPU per "node" — B200
// restatement of moesim::select_pilots / rbd_dispatch / rbd_combine
// (/root/reference/proj/src/rbd.cpp:26-358) with node_of[w] = w.
//
// A token routed to several experts on one destination GPU crosses NVLink
// once.  Per source rank:
//   groups   copies grouped by (token, destination rank), ordered (token asc,
//            dest asc) — the reference's std::map key order (rbd.cpp:35-43)
//   pilots   one Rng(salt_seed(seed, w, 0)).below(|group|) draw per group in
//            that order picks the pilot among the members in packed order
//            (rbd.cpp:45-51).  Group g uses the g-th xoshiro256** output: a
//            chunked jump-ahead (GF(2) matrix powers of the state transition)
//            lets every CTA start its 256-group chunk in parallel.
//   pack     each group's token row once (dest-major, token order) plus one
//            24-byte descriptor per copy {row in the unique buffer at the
//            receiver, row in the receiver's grouped expert input, weight,
//            group size, member index | pilot flag}
//   expand   receiver writes every copy into its grouped (local expert,
//            source, position) row — bit-identical to pf_dispatch
//
// Two-tier form (gpus_per_node > 1, rbd.cpp:83-358 with node_of = rank /
// gpus_per_node): groups are (token, destination NODE); the row lands once
// on the pilot's owner (stage 1), which forwards it to the replicas' owners
// on the same node (stage 2, an NVLink peer store in expand) and merges the
// members' outputs by reading them from their owners (reverse stage 2).
//   merge    receiver scales the pilot's expert output by its weight and adds
//            each other member's weighted output in packed order
//            (rbd.cpp:318-336); singletons return raw
//   combine  source adds its groups in pilot order with scale 1 (merged) or
//            the pilot weight (singleton) (rbd.cpp:343-356).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "rbd.h"

namespace xmoe {

// ---------------------------------------------------------------- xoshiro256**
namespace {
__host__ __device__ inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__host__ __device__ inline uint64_t xoshiro_next(uint64_t* s) {
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// 256x256 GF(2) matrix, row-major: row i has bit j set iff out_i depends on in_j.
struct Mat {
    uint64_t r[256][4];
};

void mat_mul(const Mat& A, const Mat& B, Mat& C) {  // C = A * B
    for (int i = 0; i < 256; ++i) {
        uint64_t acc[4] = {0, 0, 0, 0};
        for (int j = 0; j < 256; ++j)
            if ((A.r[i][j >> 6] >> (j & 63)) & 1)
                for (int w = 0; w < 4; ++w) acc[w] ^= B.r[j][w];
        for (int w = 0; w < 4; ++w) C.r[i][w] = acc[w];
    }
}
}  // namespace

uint64_t salt_seed_host(uint64_t seed, uint64_t a, uint64_t b) {
    // include/moesim/rng.hpp:17-19
    return splitmix64(splitmix64(seed ^ 0x6d6f6573696d0001ULL) + splitmix64(a) * 3 + b);
}

void rng_state_from_seed(uint64_t seed, uint64_t out[4]) {
    // Rng(seed) constructor, rng.hpp:26-29
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) out[i] = x = splitmix64(x);
}

// Jump matrices J_k = T^(2^log2_chunk * 2^k), k < count, T = one xoshiro step.
void gf2_jump_tables(int log2_chunk, int count, std::vector<uint64_t>& out) {
    Mat T;
    for (int j = 0; j < 256; ++j) {  // column j = T(e_j)
        uint64_t s[4] = {0, 0, 0, 0};
        s[j >> 6] = 1ull << (j & 63);
        xoshiro_next(s);
        for (int i = 0; i < 256; ++i) {
            if (j == 0) T.r[i][0] = T.r[i][1] = T.r[i][2] = T.r[i][3] = 0;
            if ((s[i >> 6] >> (i & 63)) & 1) T.r[i][j >> 6] |= 1ull << (j & 63);
        }
    }
    Mat P = T, tmp;
    for (int c = 0; c < log2_chunk; ++c) {
        mat_mul(P, P, tmp);
        P = tmp;
    }
    out.assign(static_cast<size_t>(count) * 256 * 4, 0);
    for (int k = 0; k < count; ++k) {
        for (int i = 0; i < 256; ++i)
            for (int w = 0; w < 4; ++w) out[(static_cast<size_t>(k) * 256 + i) * 4 + w] = P.r[i][w];
        mat_mul(P, P, tmp);
        P = tmp;
    }
}

// Jump matrices J_k = T^(kRbdChunk * 2^k), T = one xoshiro step.
void rbd_jump_tables(std::vector<uint64_t>& out) {
    static_assert(kRbdChunk == 256, "chunk is 2^8 outputs");
    gf2_jump_tables(8, kRbdJumps, out);
}

// One CTA per chunk of kRbdChunk groups: jump the seed state to the chunk
// start (thread i computes output bit i of each matrix-vector product), then
// one thread steps through the chunk.
__global__ void __launch_bounds__(256) rbd_draw_kernel(uint64_t s0, uint64_t s1, uint64_t s2,
                                                      uint64_t s3, const uint64_t* __restrict__ jumps,
                                                      const int32_t* __restrict__ G_dev,
                                                      uint64_t* __restrict__ draws) {
    __shared__ uint64_t st[4];
    __shared__ uint32_t bits[8];
    const int G = *G_dev;
    const int c = blockIdx.x;
    if (c * kRbdChunk >= G) return;
    if (threadIdx.x == 0) {
        st[0] = s0;
        st[1] = s1;
        st[2] = s2;
        st[3] = s3;
    }
    __syncthreads();
    const int i = threadIdx.x;
    for (int k = 0; k < kRbdJumps && (c >> k); ++k) {
        if (!((c >> k) & 1)) continue;
        const uint64_t* row = jumps + (static_cast<size_t>(k) * 256 + i) * 4;
        const int par = (__popcll(row[0] & st[0]) + __popcll(row[1] & st[1]) +
                         __popcll(row[2] & st[2]) + __popcll(row[3] & st[3])) & 1;
        const unsigned b = __ballot_sync(0xffffffffu, par);
        if ((i & 31) == 0) bits[i >> 5] = b;
        __syncthreads();
        if (i < 4) st[i] = static_cast<uint64_t>(bits[2 * i]) | (static_cast<uint64_t>(bits[2 * i + 1]) << 32);
        __syncthreads();
    }
    if (i == 0) {
        uint64_t s[4] = {st[0], st[1], st[2], st[3]};
        const int n = min(kRbdChunk, G - c * kRbdChunk);
        for (int j = 0; j < n; ++j) draws[c * kRbdChunk + j] = xoshiro_next(s);
    }
}

// ---------------------------------------------------------------- synthetic inputs
// The reference generator on the device (rng.hpp:24-47): outputs
// [offset, offset + n) of Rng(seed)'s uniform(lo, hi) stream.  The stream is
// cut into chains of kRngChain outputs; one CTA per chain jumps the seed
// state to the chain start (GF(2) powers T^(kRngChain * 2^k), bit-parallel
// over the 256 threads) and one thread then steps through the chain.
// value = lo + (hi - lo) * ((x >> 11) * 2^-53) in fp64 (separate mul/add,
// as the reference), optionally snapped to multiples of 1/grid
// (round-half-even), stored as f64, f32 or bf16 (round to nearest even).
constexpr int kRngLog2Chain = 16;
constexpr long long kRngChain = 1LL << kRngLog2Chain;
constexpr int kRngJumps = 40;

__global__ void __launch_bounds__(256) rng_fill_kernel(uint64_t s0, uint64_t s1, uint64_t s2, uint64_t s3,
                                                      const uint64_t* __restrict__ jumps, unsigned long long offset,
                                                      long long n, double lo, double hi, double grid, int dtype,
                                                      void* __restrict__ out) {
    __shared__ uint64_t st[4];
    __shared__ uint32_t bits[8];
    const unsigned long long c = offset / kRngChain + blockIdx.x;  // global chain index
    if (threadIdx.x == 0) {
        st[0] = s0;
        st[1] = s1;
        st[2] = s2;
        st[3] = s3;
    }
    __syncthreads();
    const int i = threadIdx.x;
    for (int k = 0; k < kRngJumps && (c >> k); ++k) {
        if (!((c >> k) & 1)) continue;
        const uint64_t* row = jumps + (static_cast<size_t>(k) * 256 + i) * 4;
        const int par = (__popcll(row[0] & st[0]) + __popcll(row[1] & st[1]) + __popcll(row[2] & st[2]) +
                         __popcll(row[3] & st[3])) & 1;
        const unsigned b = __ballot_sync(0xffffffffu, par);
        if ((i & 31) == 0) bits[i >> 5] = b;
        __syncthreads();
        if (i < 4) st[i] = static_cast<uint64_t>(bits[2 * i]) | (static_cast<uint64_t>(bits[2 * i + 1]) << 32);
        __syncthreads();
    }
    if (i != 0) return;
    uint64_t s[4] = {st[0], st[1], st[2], st[3]};
    const unsigned long long g0 = c * kRngChain;                    // first output of the chain
    const unsigned long long a = g0 < offset ? offset : g0;         // first one we keep
    const unsigned long long e = min(g0 + kRngChain, offset + static_cast<unsigned long long>(n));
    for (unsigned long long q = g0; q < a; ++q) xoshiro_next(s);
    const double span = hi - lo;
    for (unsigned long long q = a; q < e; ++q) {
        const double u = static_cast<double>(xoshiro_next(s) >> 11) * 0x1.0p-53;
        double v = __dadd_rn(lo, __dmul_rn(span, u));
        if (grid > 0) v = __ddiv_rn(rint(__dmul_rn(v, grid)), grid);
        const size_t o = static_cast<size_t>(q - offset);
        if (dtype == XMOE_F64) static_cast<double*>(out)[o] = v;
        else if (dtype == XMOE_F32) static_cast<float*>(out)[o] = __double2float_rn(v);
        else static_cast<__nv_bfloat16*>(out)[o] = __double2bfloat16(v);
    }
}

static const uint64_t* rng_jumps_dev() {
    static uint64_t* d_jumps[64] = {};
    int dev = 0;
    XMOE_CUDA(cudaGetDevice(&dev));
    require(dev >= 0 && dev < 64, XMOE_ERR_CUDA, "device index out of range");
    if (!d_jumps[dev]) {  // per process and device; tables are ~320 KB
        std::vector<uint64_t> jt;
        gf2_jump_tables(kRngLog2Chain, kRngJumps, jt);
        XMOE_CUDA(cudaMalloc(&d_jumps[dev], jt.size() * sizeof(uint64_t)));
        XMOE_CUDA(cudaMemcpy(d_jumps[dev], jt.data(), jt.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    }
    return d_jumps[dev];
}

void launch_rng_uniform_state(const uint64_t s[4], unsigned long long offset, long long n, double lo, double hi,
                              double grid, int dtype, void* out, cudaStream_t st) {
    if (n <= 0) return;
    const uint64_t* jumps = rng_jumps_dev();
    const unsigned long long c0 = offset / kRngChain;
    const unsigned long long c1 = (offset + static_cast<unsigned long long>(n) - 1) / kRngChain;
    const unsigned long long chains = c1 - c0 + 1;
    require(chains < (1ull << 31) && c1 < (1ull << kRngJumps), XMOE_ERR_VALIDATION, "rng_uniform: too many outputs");
    rng_fill_kernel<<<static_cast<unsigned>(chains), 256, 0, st>>>(s[0], s[1], s[2], s[3], jumps, offset, n, lo, hi,
                                                                   grid, dtype, out);
    XMOE_LAUNCH_CHECK();
}

void launch_rng_uniform(uint64_t seed, unsigned long long offset, long long n, double lo, double hi, double grid,
                        int dtype, void* out, cudaStream_t st) {
    uint64_t s[4];
    rng_state_from_seed(seed, s);
    launch_rng_uniform_state(s, offset, n, lo, hi, grid, dtype, out, st);
}

// Host: advance a generator state by n outputs (jump tables for whole chains,
// single steps for the rest).
void rng_advance(uint64_t s[4], unsigned long long n) {
    static std::vector<uint64_t> jt;
    if (jt.empty()) gf2_jump_tables(kRngLog2Chain, kRngJumps, jt);
    const unsigned long long c = n >> kRngLog2Chain;
    for (int k = 0; k < kRngJumps && (c >> k); ++k) {
        if (!((c >> k) & 1)) continue;
        uint64_t o[4] = {0, 0, 0, 0};
        for (int i = 0; i < 256; ++i) {
            const uint64_t* row = jt.data() + (static_cast<size_t>(k) * 256 + i) * 4;
            const int par = (__builtin_popcountll(row[0] & s[0]) + __builtin_popcountll(row[1] & s[1]) +
                             __builtin_popcountll(row[2] & s[2]) + __builtin_popcountll(row[3] & s[3])) & 1;
            if (par) o[i >> 6] |= 1ull << (i & 63);
        }
        for (int w = 0; w < 4; ++w) s[w] = o[w];
    }
    for (unsigned long long q = 0; q < (n & (kRngChain - 1)); ++q) xoshiro_next(s);
}

// ---------------------------------------------------------------- groups
// Per token: number of distinct destination ranks among its kept copies
// (slot_pos is ascending packed row = ascending expert = ascending dest).
__global__ void rbd_group_count_kernel(const int32_t* __restrict__ slot_pos,
                                       const int32_t* __restrict__ expert_ids, int S, int k, int El,
                                       int32_t* __restrict__ gcount) {
    // El here = experts per NODE (node key = expert / (experts per GPU x GPUs per node))
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    int n = 0, last = -1;
    for (int j = 0; j < k; ++j) {
        const int p = slot_pos[static_cast<size_t>(t) * k + j];
        if (p < 0) break;
        const int d = expert_ids[p] / El;
        if (d != last) {
            ++n;
            last = d;
        }
    }
    gcount[t] = n;
}

// Exclusive scan of n int32 (n_dev, when given, caps n on the device);
// total -> *total.  Two launches: per-tile sums of 2048 items, then every
// tile adds the sums of the tiles before it and scans itself (8 items per
// thread, warp-shuffle and block combine).  Replaced a single-CTA scan
// (27 us for the S*k = 98K group sizes of C2 on the RBD head; ncu).
constexpr int kScanThreads = 256;
constexpr int kScanPer = 8;
constexpr int kScanTile = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(const int32_t* __restrict__ in, int n_host,
                                                                      const int32_t* __restrict__ n_dev,
                                                                      int32_t* __restrict__ bsum) {
    __shared__ int32_t ws[kScanThreads / 32];
    const int n = n_dev ? min(*n_dev, n_host) : n_host;
    const int base = blockIdx.x * kScanTile;
    int sum = 0;
    if (base < n) {
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
            const int i = base + q * kScanThreads + threadIdx.x;  // coalesced
            if (i < n) sum += in[i];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
        bsum[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(const int32_t* __restrict__ in, int n_host,
                                                                  const int32_t* __restrict__ n_dev,
                                                                  const int32_t* __restrict__ bsum,
                                                                  int32_t* __restrict__ out, int32_t* __restrict__ total) {
    __shared__ int32_t ws[kScanThreads / 32];
    __shared__ int32_t s_prefix;
    const int n = n_dev ? min(*n_dev, n_host) : n_host;
    const int base = blockIdx.x * kScanTile;
    const int last = n > 0 ? (n - 1) / kScanTile : 0;
    if (static_cast<int>(blockIdx.x) > last) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid == 0) {  // sum of the earlier tiles
        int p = 0;
        for (int b = lane; b < static_cast<int>(blockIdx.x); b += 32) p += bsum[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        if (lane == 0) s_prefix = p;
    }
    // thread t scans items base + t*kScanPer .. +kScanPer-1 (blocked, vector loads)
    int v[kScanPer];
    const int i0 = base + threadIdx.x * kScanPer;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) v[q] = (i0 + q < n) ? in[i0 + q] : 0;
    int sum = 0;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        const int x = v[q];
        v[q] = sum;
        sum += x;
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    int before = s_prefix + incl - sum;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w)
        if (w < wid) before += ws[w];
#pragma unroll
    for (int q = 0; q < kScanPer; ++q)
        if (i0 + q < n) out[i0 + q] = before + v[q];
    if (static_cast<int>(blockIdx.x) == last && threadIdx.x == kScanThreads - 1 && total)
        *total = n > 0 ? before + sum : 0;
}

static void scan_i32(const int32_t* in, int n, const int32_t* n_dev, int32_t* out, int32_t* total, int32_t* ws,
                     cudaStream_t st) {
    const int nb = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
    scan_tile_sums_kernel<<<nb, kScanThreads, 0, st>>>(in, n, n_dev, ws);
    XMOE_LAUNCH_CHECK();
    scan_tiles_kernel<<<nb, kScanThreads, 0, st>>>(in, n, n_dev, ws, out, total);
    XMOE_LAUNCH_CHECK();
}

// Per token: emit its groups (gid = gbase[t] + j) with the drawn pilot.
__global__ void rbd_group_fill_kernel(const int32_t* __restrict__ slot_pos,
                                      const int32_t* __restrict__ expert_ids, int S, int k, int El,
                                      int El_rank, const int32_t* __restrict__ gbase,
                                      const uint64_t* __restrict__ draws, RbdGroups g,
                                      int32_t* __restrict__ flags) {
    // groups: runs of equal node (El = experts per node); a group lands on
    // its pilot's owner (rbd.cpp:135-150: stage 1 goes to the pilot's worker)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    int gid = gbase[t];
    int j = 0;
    while (j < k) {
        const int p0 = slot_pos[static_cast<size_t>(t) * k + j];
        if (p0 < 0) break;
        const int d = expert_ids[p0] / El;
        int n = 1;
        while (j + n < k) {
            const int p = slot_pos[static_cast<size_t>(t) * k + j + n];
            if (p < 0 || expert_ids[p] / El != d) break;
            ++n;
        }
        // Rng::below(n) (rng.hpp:49-54): reject the top partial bucket
        const uint64_t x = draws[gid];
        const uint64_t limit = ~0ull - (~0ull % static_cast<uint64_t>(n) + 1) % static_cast<uint64_t>(n);
        if (x > limit) atomicExch(flags, 1);  // probability ~n/2^64: reported, not replayed
        const int pick = static_cast<int>(x % static_cast<uint64_t>(n));
        const int pilot = slot_pos[static_cast<size_t>(t) * k + j + pick];
        g.token[gid] = t;
        g.dest[gid] = expert_ids[pilot] / El_rank;
        g.first_slot[gid] = j;
        g.n[gid] = n;
        g.pilot[gid] = pilot;
        (void)d;
        ++gid;
        j += n;
    }
}

// Position of every group in the dest-sorted order -> per-dest index u and
// the group's first descriptor.  perm/ptr come from the stable CSR by dest.
__global__ void rbd_group_pos_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ G_dev,
                                     const RbdGroups g, int32_t* __restrict__ nsorted) {
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= *G_dev) return;
    const int gid = perm[pos];
    g.pos[gid] = pos;
    nsorted[pos] = g.n[gid];
}

__device__ __forceinline__ int rbd_chunk_t0(int c, int S, int C) { return chunk_t0(c, S, C); }

// first descriptor (my order) of sorted position p; p == G gives the total
__device__ __forceinline__ int rbd_coff_at(const int32_t* coff, const int32_t* nsorted, int G, int p) {
    return p < G ? coff[p] : (G > 0 ? coff[G - 1] + nsorted[G - 1] : 0);
}

// Sender side, before the count all-gather: chunk boundaries inside every
// dest segment (binary search on the token; segments are token-ordered) and
// the groups / copies per (dest, chunk).
__global__ void rbd_chunk_counts_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ G_dev,
                                        const int32_t* __restrict__ gtoken, const int32_t* __restrict__ dptr,
                                        const int32_t* __restrict__ coff, const int32_t* __restrict__ nsorted,
                                        int W, int S, int C, int32_t* __restrict__ gpos,
                                        int32_t* __restrict__ gd_own) {
    const int G = *G_dev;
    for (int idx = threadIdx.x; idx < W * (C + 1); idx += blockDim.x) {
        const int d = idx / (C + 1), c = idx % (C + 1);
        const int b = dptr[d], n = dptr[d + 1] - b;
        int v;
        if (c == 0) v = 0;
        else if (c == C) v = n;
        else {
            const int t0 = rbd_chunk_t0(c, S, C);
            int lo = 0, hi = n;
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (gtoken[perm[b + m]] < t0) lo = m + 1;
                else hi = m;
            }
            v = lo;
        }
        gpos[idx] = v;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < W * C; idx += blockDim.x) {
        const int d = idx / C, c = idx % C;
        const int p0 = dptr[d] + gpos[d * (C + 1) + c], p1 = dptr[d] + gpos[d * (C + 1) + c + 1];
        gd_own[idx] = p1 - p0;  // groups
        gd_own[W * C + idx] = rbd_coff_at(coff, nsorted, G, p1) - rbd_coff_at(coff, nsorted, G, p0);  // copies
    }
}

// Offsets, all on the device (no host sync).  Receivers keep groups and
// descriptors in (chunk, source, sender order):
//   ru[d][c]  first row of my chunk-c groups in d's merged-row buffer
//   rd[d][c]  first slot of my chunk-c descriptors in d's descriptor buffer
//   cs[d][c]  first descriptor of my (d, c) segment in my own order
//   rx[.][c]  what I receive in chunk c: group base / count, descriptor base / count
__global__ void rbd_offsets_kernel(const int32_t* __restrict__ gd_all, int W, int C, int me,
                                   const int32_t* __restrict__ gpos, const int32_t* __restrict__ dptr,
                                   const int32_t* __restrict__ coff, const int32_t* __restrict__ nsorted,
                                   const int32_t* __restrict__ G_dev, int32_t* __restrict__ ru,
                                   int32_t* __restrict__ rd, int32_t* __restrict__ cs,
                                   int32_t* __restrict__ rx) {
    auto GD = [&](int s, int which, int d, int c) {
        return gd_all[((static_cast<size_t>(s) * 2 + which) * W + d) * C + c];
    };
    const int G = *G_dev;
    for (int idx = threadIdx.x; idx < W * C; idx += blockDim.x) {
        const int d = idx / C, c = idx % C;
        int g = 0, q = 0;
        for (int c2 = 0; c2 < c; ++c2)
            for (int s = 0; s < W; ++s) {
                g += GD(s, 0, d, c2);
                q += GD(s, 1, d, c2);
            }
        for (int s = 0; s < me; ++s) {
            g += GD(s, 0, d, c);
            q += GD(s, 1, d, c);
        }
        ru[idx] = g;
        rd[idx] = q;
        cs[idx] = rbd_coff_at(coff, nsorted, G, dptr[d] + gpos[d * (C + 1) + c]);
    }
    if (threadIdx.x == 0) {
        int gb = 0, qb = 0;
        for (int c = 0; c < C; ++c) {
            int g = 0, q = 0;
            for (int s = 0; s < W; ++s) {
                g += GD(s, 0, me, c);
                q += GD(s, 1, me, c);
            }
            rx[c] = gb;
            rx[C + c] = g;
            rx[2 * C + c] = qb;
            rx[3 * C + c] = q;
            gb += g;
            qb += q;
        }
    }
}

// Token-major sender pack: one warp per token of chunk c loads the token's
// row once and stores it to each of its (token, dest) groups' pilot slot;
// lane l < kept(t) writes slot l's descriptor.  Same bytes as the
// group-major pack, k-fold fewer dependent row loads per warp.
constexpr int kPackVec = 8;  // int4 per lane per pass (4 KB rows in one pass)
__global__ void __launch_bounds__(512) rbd_pack_tokens_kernel(
    const char* __restrict__ x, int row_bytes, int S, int C, int c, int k, int El,
    const int32_t* __restrict__ slot_pos, const int32_t* __restrict__ expert_ids,
    const int32_t* __restrict__ dest_row, const double* __restrict__ cw, const int32_t* __restrict__ gbase,
    const int32_t* __restrict__ gcount, const RbdGroups g, const int32_t* __restrict__ dptr,
    const int32_t* __restrict__ coff, const int32_t* __restrict__ gpos, const int32_t* __restrict__ ru,
    const int32_t* __restrict__ rd, const int32_t* __restrict__ cs, char* const* __restrict__ recv_u_tab,
    RbdDesc* const* __restrict__ desc_tab, int gpn) {
    const int lane = threadIdx.x & 31;
    const bool vec = (row_bytes & 15) == 0;  // else 8-byte rows (F64, odd model_dim)
    const int t_beg = rbd_chunk_t0(c, S, C), t_end = rbd_chunk_t0(c + 1, S, C);
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int nvec = row_bytes >> 4;
    for (long long tt = t_beg + warp; tt < t_end; tt += nwarps) {
        const int t = static_cast<int>(tt);
        const int4* src = reinterpret_cast<const int4*>(x + static_cast<size_t>(t) * row_bytes);
        int4 v[kPackVec];
#pragma unroll
        for (int q = 0; q < kPackVec; ++q) {
            const int col = lane + 32 * q;
            v[q] = vec && col < nvec ? ld_nc_v4(src + col) : make_int4(0, 0, 0, 0);
        }
        const int ng = gcount[t], b = gbase[t];
        // lane j < ng: group j of the token (dest ascending)
        unsigned long long dst = 0;
        int gn = 0, gpilot = -1, gdesc = 0, gu = 0, gd = 0;
        if (lane < ng) {
            const int gid = b + lane;
            gd = g.dest[gid];
            gn = g.n[gid];
            gpilot = g.pilot[gid];
            const int pos = g.pos[gid];
            gu = ru[gd * C + c] + pos - dptr[gd] - gpos[gd * (C + 1) + c];
            gdesc = rd[gd * C + c] + (coff[pos] - cs[gd * C + c]);
            dst = reinterpret_cast<unsigned long long>(recv_u_tab[gd] +
                                                       static_cast<size_t>(dest_row[gpilot]) * row_bytes);
        }
        // lane l < kept(t): descriptor of slot l (groups are runs of equal dest)
        const int p = lane < k ? slot_pos[static_cast<size_t>(t) * k + lane] : -1;
        const int owner = p >= 0 ? expert_ids[p] / El : -1;
        const int dl = p >= 0 ? owner / gpn : -1;  // group key: the member's node
        const int dprev = __shfl_up_sync(0xffffffffu, dl, 1);
        const unsigned starts = __ballot_sync(0xffffffffu, p >= 0 && (lane == 0 || dl != dprev));
        const unsigned le = starts & (0xffffffffu >> (31 - lane));
        const int gj = __popc(le) - 1;
        const int m = le ? lane - (31 - __clz(le)) : 0;
        const int jd = gj < 0 ? 0 : gj;
        const int n_j = __shfl_sync(0xffffffffu, gn, jd);
        const int pil_j = __shfl_sync(0xffffffffu, gpilot, jd);
        const int desc_j = __shfl_sync(0xffffffffu, gdesc, jd);
        const int u_j = __shfl_sync(0xffffffffu, gu, jd);
        const int d_j = __shfl_sync(0xffffffffu, gd, jd);
        if (p >= 0) {
            RbdDesc dd;
            dd.u = u_j;
            dd.dest_row = dest_row[p];
            dd.w = cw[p];
            dd.n = n_j;
            dd.member = m | (p == pil_j ? kRbdPilotFlag : 0) | (owner << kRbdOwnerShift);
            desc_tab[d_j][desc_j + m] = dd;
        }
        if (!vec) {
            const long long* s8 = reinterpret_cast<const long long*>(src);
            for (int j = 0; j < ng; ++j) {
                long long* d8 = reinterpret_cast<long long*>(__shfl_sync(0xffffffffu, dst, j));
                for (int q = lane; q < (row_bytes >> 3); q += 32) d8[q] = s8[q];
            }
            continue;
        }
        for (int base = 0; base < nvec; base += 32 * kPackVec) {
            if (base > 0) {
#pragma unroll
                for (int q = 0; q < kPackVec; ++q) {
                    const int col = base + lane + 32 * q;
                    v[q] = col < nvec ? ld_nc_v4(src + col) : make_int4(0, 0, 0, 0);
                }
            }
            for (int j = 0; j < ng; ++j) {
                int4* d = reinterpret_cast<int4*>(__shfl_sync(0xffffffffu, dst, j));
#pragma unroll
                for (int q = 0; q < kPackVec; ++q) {
                    const int col = base + lane + 32 * q;
                    if (col < nvec) st_na_v4(d + col, v[q]);
                }
            }
        }
    }
    __threadfence_system();
}

// Receiver expand: every replica copies its group's row from the pilot's
// slot (where the sender put it) into its own grouped slot; records each
// group's first descriptor for the merge.
__global__ void __launch_bounds__(256) rbd_expand_kernel(char* const* __restrict__ recv_tab,
                                                         int row_bytes, const RbdDesc* __restrict__ desc,
                                                         const int32_t* __restrict__ rx, int C, int ck,
                                                         const char* __restrict__ grouped,
                                                         int32_t* __restrict__ gstart,
                                                         int32_t* __restrict__ a_idx) {
    const int dbeg = rx[2 * C + ck], dend = dbeg + rx[3 * C + ck];
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long c = dbeg + warp; c < dend; c += nwarps) {
        const RbdDesc dd = desc[c];
        const int m = dd.member & kRbdMemberMask;
        if (lane == 0 && m == 0) gstart[dd.u] = static_cast<int>(c);
        if (a_idx) {  // gather mode: GEMM1 reads every copy's row through a_idx
            if (lane == 0) {
                int prow = dd.dest_row;
                for (int q = 0; q < dd.n; ++q) {
                    const RbdDesc pq = desc[c - m + q];
                    if (pq.member & kRbdPilotFlag) prow = pq.dest_row;
                }
                a_idx[dd.dest_row] = prow;
            }
            continue;
        }
        if (dd.member & kRbdPilotFlag) continue;  // already in place
        int prow = dd.dest_row;
        for (int q = 0; q < dd.n; ++q) {
            const RbdDesc pq = desc[c - m + q];
            if (pq.member & kRbdPilotFlag) prow = pq.dest_row;
        }
        // the pilot landed here; a replica owned by another GPU of the node
        // gets its row over NVLink (stage 2, rbd.cpp:178-233)
        const char* s = grouped + static_cast<size_t>(prow) * row_bytes;
        char* o = recv_tab[dd.member >> kRbdOwnerShift] + static_cast<size_t>(dd.dest_row) * row_bytes;
        if ((row_bytes & 15) == 0) {
            for (int v = lane; v < (row_bytes >> 4); v += 32)
                st_na_v4(reinterpret_cast<int4*>(o) + v, reinterpret_cast<const int4*>(s)[v]);
        } else {
            for (int v = lane; v < (row_bytes >> 3); v += 32)
                reinterpret_cast<long long*>(o)[v] = reinterpret_cast<const long long*>(s)[v];
        }
    }
}

// Receiver merge (rbd.cpp:318-336): one warp per received group.
template <typename T>
__global__ void __launch_bounds__(256) rbd_merge_kernel(const char* const* __restrict__ eout_tab, int H,
                                                        const RbdDesc* __restrict__ desc,
                                                        const int32_t* __restrict__ gstart,
                                                        const int32_t* __restrict__ rx, int C, int ck,
                                                        T* __restrict__ back_u) {
    const int ubeg = rx[ck], uend = ubeg + rx[C + ck];
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long u = ubeg + warp; u < uend; u += nwarps) {
        const int c0 = gstart[u];
        const int n = desc[c0].n;
        T* out = back_u + static_cast<size_t>(u) * H;
        auto row_of = [&](const RbdDesc& d) {
            return reinterpret_cast<const T*>(eout_tab[d.member >> kRbdOwnerShift]) + static_cast<size_t>(d.dest_row) * H;
        };
        if (n == 1) {  // singleton: raw row
            const T* y = row_of(desc[c0]);
            for (int h = lane; h < H; h += 32) out[h] = y[h];
            continue;
        }
        int pm = 0;
        for (int m = 0; m < n; ++m)
            if (desc[c0 + m].member & kRbdPilotFlag) pm = m;
        const RbdDesc pd = desc[c0 + pm];
        for (int h = lane; h < H; h += 32) {
            if constexpr (sizeof(T) == 8) {
                double acc = __dmul_rn(static_cast<double>(row_of(pd)[h]), pd.w);
                for (int m = 0; m < n; ++m) {
                    if (m == pm) continue;
                    const RbdDesc md = desc[c0 + m];
                    acc = __dadd_rn(acc, __dmul_rn(md.w, static_cast<double>(row_of(md)[h])));
                }
                out[h] = static_cast<T>(acc);
            } else if constexpr (sizeof(T) == 4) {  // F32: the reference's scale / axpy order, fp64 accumulation
                double acc = __dmul_rn(static_cast<double>(row_of(pd)[h]), pd.w);
                for (int m = 0; m < n; ++m) {
                    if (m == pm) continue;
                    const RbdDesc md = desc[c0 + m];
                    acc = __dadd_rn(acc, __dmul_rn(md.w, static_cast<double>(row_of(md)[h])));
                }
                out[h] = static_cast<T>(acc);
            } else {
                float acc = __bfloat162float(row_of(pd)[h]) * static_cast<float>(pd.w);
                for (int m = 0; m < n; ++m) {
                    if (m == pm) continue;
                    const RbdDesc md = desc[c0 + m];
                    acc = fmaf(static_cast<float>(md.w), __bfloat162float(row_of(md)[h]), acc);
                }
                out[h] = __float2bfloat16_rn(acc);
            }
        }
    }
}

// Source combine (rbd.cpp:343-356): per token, its groups in pilot order;
// each merged row is read straight from its landing rank's back_u.
template <typename T>
__global__ void __launch_bounds__(256) rbd_combine_kernel(const char* const* __restrict__ back_tab, int H,
                                                          int S, const int32_t* __restrict__ gbase,
                                                          const int32_t* __restrict__ gcount,
                                                          const RbdGroups g, const int32_t* __restrict__ ru,
                                                          const int32_t* __restrict__ gpos, int C, int ck,
                                                          const int32_t* __restrict__ dptr,
                                                          const double* __restrict__ cw,
                                                          const T* __restrict__ addend, T* __restrict__ out) {
    const int t = rbd_chunk_t0(ck, S, C) + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= rbd_chunk_t0(ck + 1, S, C)) return;
    const int b = gbase[t], n = gcount[t];
    // groups of a token are few (<= min(k, W)): order them by pilot packed row
    int order[32];
    const int nn = n < 32 ? n : 32;
    for (int i = 0; i < nn; ++i) {
        int q = i;
        const int pi = g.pilot[b + i];
        while (q > 0 && g.pilot[b + order[q - 1]] > pi) {
            order[q] = order[q - 1];
            --q;
        }
        order[q] = i;
    }
    const T* rowp[32];
    for (int i = 0; i < nn; ++i) {
        const int gid = b + order[i];
        const int d = g.dest[gid];
        rowp[i] = reinterpret_cast<const T*>(back_tab[d]) +
                  static_cast<size_t>(ru[d * C + ck] + g.pos[gid] - dptr[d] - gpos[d * (C + 1) + ck]) * H;
    }
    for (int h = lane; h < H; h += 32) {
        if constexpr (sizeof(T) == 8) {
            double acc = 0.0;
            for (int i = 0; i < nn; ++i) {
                const int gid = b + order[i];
                const double sc = g.n[gid] > 1 ? 1.0 : cw[g.pilot[gid]];
                acc = __dadd_rn(acc, __dmul_rn(sc, static_cast<double>(rowp[i][h])));
            }
            if (addend) acc = __dadd_rn(acc, static_cast<double>(addend[static_cast<size_t>(t) * H + h]));
            out[static_cast<size_t>(t) * H + h] = static_cast<T>(acc);
        } else if constexpr (sizeof(T) == 4) {  // F32: fp64 accumulation, one rounding
            double acc = 0.0;
            for (int i = 0; i < nn; ++i) {
                const int gid = b + order[i];
                const double sc = g.n[gid] > 1 ? 1.0 : cw[g.pilot[gid]];
                acc = __dadd_rn(acc, __dmul_rn(sc, static_cast<double>(rowp[i][h])));
            }
            if (addend) acc = __dadd_rn(acc, static_cast<double>(addend[static_cast<size_t>(t) * H + h]));
            out[static_cast<size_t>(t) * H + h] = static_cast<T>(acc);
        } else {
            float acc = 0.f;
            for (int i = 0; i < nn; ++i) {
                const int gid = b + order[i];
                const float sc = g.n[gid] > 1 ? 1.f : static_cast<float>(cw[g.pilot[gid]]);
                acc = fmaf(sc, __bfloat162float(rowp[i][h]), acc);
            }
            if (addend) acc += __bfloat162float(addend[static_cast<size_t>(t) * H + h]);
            out[static_cast<size_t>(t) * H + h] = __float2bfloat16_rn(acc);
        }
    }
}

// BF16 merge, vectorised: one warp per (received group, 512-column segment);
// lane m < n holds member m's row and weight, the pilot is applied first,
// every row moves 16 bytes per lane, fp32 math.
__global__ void __launch_bounds__(256) rbd_merge_bf16_kernel(const char* const* __restrict__ eout_tab, int H,
                                                             const RbdDesc* __restrict__ desc,
                                                             const int32_t* __restrict__ gstart,
                                                             const int32_t* __restrict__ rx, int C, int ck,
                                                             __nv_bfloat16* __restrict__ back_u) {
    const int ubeg = rx[ck], ngroups = rx[C + ck];
    const int nseg = (H + 511) / 512;
    const int lane = threadIdx.x & 31;
    const int nchunk = H >> 3;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long item = warp; item < static_cast<long long>(ngroups) * nseg; item += nwarps) {
        const int u = ubeg + static_cast<int>(item / nseg), seg = static_cast<int>(item % nseg);
        const int c0 = gstart[u];
        const int n = desc[c0].n;
        const __nv_bfloat16* my_row = nullptr;
        float my_w = 0.f;
        int is_p = 0;
        if (lane < n) {
            const RbdDesc md = desc[c0 + lane];
            my_row = reinterpret_cast<const __nv_bfloat16*>(eout_tab[md.member >> kRbdOwnerShift]) +
                     static_cast<size_t>(md.dest_row) * H;
            my_w = static_cast<float>(md.w);
            is_p = (md.member & kRbdPilotFlag) ? 1 : 0;
        }
        const unsigned pm = __ballot_sync(0xffffffffu, is_p);
        const int pl = pm ? __ffs(pm) - 1 : 0;
        const int cbeg = seg * 64, cend = min(nchunk, cbeg + 64);
        int4* dst = reinterpret_cast<int4*>(back_u + static_cast<size_t>(u) * H);
        for (int cc = cbeg; cc < cend; cc += 32) {
            const int c = cc + lane;
            const bool ok = c < cend;
            float acc[8];
            {
                const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), pl));
                const float wp = n == 1 ? 1.f : __shfl_sync(0xffffffffu, my_w, pl);
                const int4 v = ok ? ld_nc_v4(reinterpret_cast<const int4*>(r) + c) : make_int4(0, 0, 0, 0);
                if (n == 1) {  // singleton: raw row (rbd.cpp:323-325)
                    if (ok) dst[c] = v;
                    continue;
                }
                const uint32_t q[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                       static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[2 * i] = bf16_lo(q[i]) * wp;
                    acc[2 * i + 1] = bf16_hi(q[i]) * wp;
                }
            }
            for (int m = 0; m < n; ++m) {
                if (m == pl) continue;
                const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), m));
                const float wm = __shfl_sync(0xffffffffu, my_w, m);
                const int4 v = ok ? ld_nc_v4(reinterpret_cast<const int4*>(r) + c) : make_int4(0, 0, 0, 0);
                const uint32_t q[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                       static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[2 * i] = fmaf(wm, bf16_lo(q[i]), acc[2 * i]);
                    acc[2 * i + 1] = fmaf(wm, bf16_hi(q[i]), acc[2 * i + 1]);
                }
            }
            if (ok) {
                int4 o;
                o.x = static_cast<int>(pack_bf16(acc[0], acc[1]));
                o.y = static_cast<int>(pack_bf16(acc[2], acc[3]));
                o.z = static_cast<int>(pack_bf16(acc[4], acc[5]));
                o.w = static_cast<int>(pack_bf16(acc[6], acc[7]));
                dst[c] = o;
            }
        }
    }
}

// BF16 source combine, vectorised: one warp per (token, 512-column segment).
// Lane i < #groups resolves group i's merged-row address (peer or local);
// the warp then permutes them into pilot order and streams the rows.
__global__ void __launch_bounds__(1024) rbd_combine_bf16_kernel(
    const char* const* __restrict__ back_tab, int H, int S, const int32_t* __restrict__ gbase,
    const int32_t* __restrict__ gcount, const RbdGroups g, const int32_t* __restrict__ ru,
    const int32_t* __restrict__ gpos, int C, int ck, const int32_t* __restrict__ dptr,
    const double* __restrict__ cw, const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ out) {
    const int nseg = (H + 511) / 512;
    const int t0 = rbd_chunk_t0(ck, S, C), nt = rbd_chunk_t0(ck + 1, S, C) - t0;
    const int lane = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    // grid-stride: the whole-SM launch of the SM partition has fewer warps than items
    for (long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
         gw < static_cast<long long>(nt) * nseg; gw += nw) {
    const int t = t0 + static_cast<int>(gw / nseg), seg = static_cast<int>(gw % nseg);
    const int b = gbase[t], n = min(gcount[t], 32);
    int key = 0x7fffffff;
    unsigned long long rp = 0;
    float sc = 0.f;
    if (lane < n) {
        const int gid = b + lane;
        const int d = g.dest[gid];
        key = g.pilot[gid];
        rp = reinterpret_cast<unsigned long long>(
            reinterpret_cast<const __nv_bfloat16*>(back_tab[d]) +
            static_cast<size_t>(ru[d * C + ck] + g.pos[gid] - dptr[d] - gpos[d * (C + 1) + ck]) * H);
        sc = g.n[gid] > 1 ? 1.f : static_cast<float>(cw[key]);
    }
    int rank = 0;  // position of my group in pilot order (rbd.cpp:343-356)
    for (int j = 0; j < n; ++j) rank += __shfl_sync(0xffffffffu, key, j) < key;
    int my_src = 0;  // lane o gathers the group of rank o
    for (int o = 0; o < n; ++o) {
        const unsigned bm = __ballot_sync(0xffffffffu, lane < n && rank == o);
        if (lane == o) my_src = __ffs(bm) - 1;
    }
    const unsigned long long orp = __shfl_sync(0xffffffffu, rp, my_src);
    const float osc = __shfl_sync(0xffffffffu, sc, my_src);
    const int nchunk = H >> 3;
    const int cbeg = seg * 64, cend = min(nchunk, cbeg + 64);
    for (int cc = cbeg; cc < cend; cc += 32) {
        const int c = cc + lane;
        const bool ok = c < cend;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int o = 0; o < n; ++o) {
            const int4* p = reinterpret_cast<const int4*>(__shfl_sync(0xffffffffu, orp, o));
            const float s = __shfl_sync(0xffffffffu, osc, o);
            const int4 v = ok ? ld_nc_v4(p + c) : make_int4(0, 0, 0, 0);
            const uint32_t q[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                   static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[2 * i] = fmaf(s, bf16_lo(q[i]), acc[2 * i]);
                acc[2 * i + 1] = fmaf(s, bf16_hi(q[i]), acc[2 * i + 1]);
            }
        }
        if (!ok) continue;
        if (addend) {
            const int4 v = ld_nc_v4(reinterpret_cast<const int4*>(addend + static_cast<size_t>(t) * H) + c);
            const uint32_t q[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                   static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[2 * i] += bf16_lo(q[i]);
                acc[2 * i + 1] += bf16_hi(q[i]);
            }
        }
        int4 o;
        o.x = static_cast<int>(pack_bf16(acc[0], acc[1]));
        o.y = static_cast<int>(pack_bf16(acc[2], acc[3]));
        o.z = static_cast<int>(pack_bf16(acc[4], acc[5]));
        o.w = static_cast<int>(pack_bf16(acc[6], acc[7]));
        st_na_v4(reinterpret_cast<int4*>(out + static_cast<size_t>(t) * H) + c, o);
    }
    }
}

// ---------------------------------------------------------------- byte ledger counts
// Device counters behind the byte ledger of the last forward (ledger.cpp):
//   out[0]                       (token, destination rank != me) groups: the rows
//                                the redundancy bypass sends off-rank (rbd.cpp:427-442)
//   out[1 + L]                   pilots landing at L (stage-1 rows, merged rows home)
//   out[1 + W + L]               ... of groups with replicas (their weight rides along)
//   out[1 + 2W + L]              replicas whose descriptors ride to L
//   out[1 + 3W + L * W + o]      replicas forwarded by L to owner o (stage 2)
// Block-level counts in shared memory, one global atomic per nonzero counter.
__global__ void __launch_bounds__(256) ledger_counts_kernel(const int32_t* __restrict__ slot_pos, int S, int k,
                                                            const int32_t* __restrict__ expert_ids, int El, int me,
                                                            RbdGroups g, const int32_t* __restrict__ G_dev, int W,
                                                            unsigned long long* __restrict__ out) {
    extern __shared__ unsigned int cnt[];
    const int ncnt = 1 + 3 * W + W * W;
    for (int i = threadIdx.x; i < ncnt; i += blockDim.x) cnt[i] = 0u;
    __syncthreads();
    const int G = (G_dev && g.pilot) ? *G_dev : 0;
    const int n_items = S > G ? S : G;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x) {
        if (i < S) {  // distinct off-rank destinations of token i (slots ascending = dests ascending)
            int last = -1, nd = 0;
            for (int j = 0; j < k; ++j) {
                const int p = slot_pos[static_cast<size_t>(i) * k + j];
                if (p < 0) break;
                const int d = expert_ids[p] / El;
                if (d != me && d != last) ++nd;
                last = d;
            }
            if (nd) atomicAdd(&cnt[0], static_cast<unsigned>(nd));
        }
        if (i < G) {
            const int L = g.dest[i], n = g.n[i], t = g.token[i], f = g.first_slot[i], pl = g.pilot[i];
            atomicAdd(&cnt[1 + L], 1u);
            if (n > 1) atomicAdd(&cnt[1 + W + L], 1u);
            for (int m = 0; m < n; ++m) {
                const int p = slot_pos[static_cast<size_t>(t) * k + f + m];
                if (p == pl) continue;
                atomicAdd(&cnt[1 + 2 * W + L], 1u);
                atomicAdd(&cnt[1 + 3 * W + L * W + expert_ids[p] / El], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ncnt; i += blockDim.x)
        if (cnt[i]) atomicAdd(&out[i], static_cast<unsigned long long>(cnt[i]));
}

void launch_ledger_counts(const int32_t* slot_pos, int S, int k, const int32_t* expert_ids, int El, int me,
                          const RbdWork* wk, int W, unsigned long long* out, cudaStream_t st) {
    const int ncnt = 1 + 3 * W + W * W;
    require(ncnt * 4 <= 48 * 1024, XMOE_ERR_VALIDATION, "ledger counters: world too large");
    XMOE_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long) * ncnt, st));
    RbdGroups g{};
    const int32_t* G_dev = nullptr;
    long long items = S;
    if (wk) {
        g = wk->g;
        G_dev = wk->G_dev;
        items = std::max<long long>(S, static_cast<long long>(S) * k);
    }
    if (items == 0) return;
    const long long blocks = std::min<long long>((items + 255) / 256, 4LL * kNumSMs);
    ledger_counts_kernel<<<static_cast<int>(blocks), 256, sizeof(unsigned) * ncnt, st>>>(
        slot_pos, S, k, expert_ids, El, me, g, G_dev, W, out);
    XMOE_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- launchers
static int warp_grid(long long items) {
    const long long b = (items + 7) / 8;
    return static_cast<int>(b < 1 ? 1 : (b < 8 * kNumSMs ? b : 8 * kNumSMs));
}

void launch_rbd_groups(const int32_t* slot_pos, const int32_t* expert_ids, int S, int k, int El,
                       const uint64_t state[4], const uint64_t* jumps, RbdWork& wk, cudaStream_t st) {
    if (S == 0) {
        XMOE_CUDA(cudaMemsetAsync(wk.G_dev, 0, sizeof(int32_t), st));
        return;
    }
    const int El_node = El * wk.gpn;  // group key: the copy's node
    rbd_group_count_kernel<<<ceil_div(S, 256), 256, 0, st>>>(slot_pos, expert_ids, S, k, El_node, wk.gcount);
    XMOE_LAUNCH_CHECK();
    scan_i32(wk.gcount, S, nullptr, wk.gbase, wk.G_dev, wk.scan_ws, st);
    const long long max_groups = static_cast<long long>(S) * k;
    rbd_draw_kernel<<<ceil_div(max_groups, kRbdChunk), 256, 0, st>>>(
        state[0], state[1], state[2], state[3], jumps, wk.G_dev, wk.draws);
    XMOE_LAUNCH_CHECK();
    rbd_group_fill_kernel<<<ceil_div(S, 256), 256, 0, st>>>(slot_pos, expert_ids, S, k, El_node, El, wk.gbase,
                                                             wk.draws, wk.g, wk.flags);
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_sort(int W, long long max_groups, RbdWork& wk, cudaStream_t st) {
    // stable bucket of groups by destination (groups are generated in
    // (token, dest) order, so each dest segment stays in token order)
    launch_stable_csr_dev(wk.g.dest, wk.G_dev, static_cast<int>(max_groups), W, wk.dptr, wk.perm,
                          wk.csr_ws, st);
    if (max_groups == 0) return;  // empty sequence: dptr zeroed above
    rbd_group_pos_kernel<<<ceil_div(max_groups, 256), 256, 0, st>>>(wk.perm, wk.G_dev, wk.g, wk.nsorted);
    XMOE_LAUNCH_CHECK();
    scan_i32(wk.nsorted, static_cast<int>(max_groups), wk.G_dev, wk.coff, nullptr, wk.scan_ws, st);
}

void launch_rbd_chunk_counts(int W, int S, RbdWork& wk, cudaStream_t st) {
    rbd_chunk_counts_kernel<<<1, 256, 0, st>>>(wk.perm, wk.G_dev, wk.g.token, wk.dptr, wk.coff, wk.nsorted, W,
                                               S, wk.C, wk.gpos, wk.gd_own);
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_offsets(const int32_t* gd_all, int W, int me, RbdWork& wk, cudaStream_t st) {
    rbd_offsets_kernel<<<1, 256, 0, st>>>(gd_all, W, wk.C, me, wk.gpos, wk.dptr, wk.coff, wk.nsorted, wk.G_dev,
                                          wk.ru, wk.rd, wk.cs, wk.rx);
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_pack(const void* x, int row_bytes, const RbdWork& wk, int W, int c, long long max_groups,
                     const int32_t* slot_pos, int k, const int32_t* dest_row, const double* cw,
                     char* const* recv_u_tab, RbdDesc* const* desc_tab, cudaStream_t st, int S,
                     const int32_t* expert_ids, int El) {
    (void)W;
    (void)max_groups;
    require((row_bytes & 7) == 0 && k <= 32 && expert_ids, XMOE_ERR_VALIDATION,
            "rbd pack needs 8-byte rows, top_k <= 32");
    const int nt = chunk_t0(c + 1, S, wk.C) - chunk_t0(c, S, wk.C);
    if (nt == 0) return;
    int tg = warp_grid(nt), threads = 256;
    size_t smem = 0;
    if (g_copy_fat > 0) {  // whole-SM blocks of the SM partition (kernels.cuh g_copy_fat)
        static bool attr = false;
        if (!attr) {
            XMOE_CUDA(cudaFuncSetAttribute(rbd_pack_tokens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kFatSmemBytes));
            attr = true;
        }
        tg = g_copy_fat;
        threads = 512;
        smem = kFatSmemBytes;
    } else if (g_copy_blocks > 0 && tg > g_copy_blocks) {
        tg = g_copy_blocks;
    }
    rbd_pack_tokens_kernel<<<tg, threads, smem, st>>>(static_cast<const char*>(x), row_bytes, S, wk.C, c, k, El, slot_pos,
                                               expert_ids, dest_row, cw, wk.gbase, wk.gcount, wk.g, wk.dptr, wk.coff,
                                               wk.gpos, wk.ru, wk.rd, wk.cs, recv_u_tab, desc_tab, wk.gpn);
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_expand(int row_bytes, const RbdDesc* desc, const RbdWork& wk, int c, long long max_desc,
                       void* grouped, char* const* recv_tab, int32_t* gstart, cudaStream_t st, int32_t* a_idx) {
    int grid = warp_grid(max_desc / wk.C + 1);
    if (g_copy_blocks > 0 && grid > g_copy_blocks) grid = g_copy_blocks;
    rbd_expand_kernel<<<grid, 256, 0, st>>>(recv_tab, row_bytes, desc, wk.rx, wk.C, c,
                                            static_cast<const char*>(grouped), gstart, a_idx);
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_merge(int dtype, const char* const* eout_tab, int H, const RbdDesc* desc, const int32_t* gstart,
                      const RbdWork& wk, int c, long long max_groups, void* back_u, cudaStream_t st) {
    const long long per = max_groups / wk.C + 1;
    auto cap = [](int g) { return g_copy_blocks > 0 && g > g_copy_blocks ? g_copy_blocks : g; };
    if (dtype == XMOE_F64)
        rbd_merge_kernel<double><<<cap(warp_grid(per)), 256, 0, st>>>(eout_tab, H, desc, gstart, wk.rx, wk.C, c,
                                                                     static_cast<double*>(back_u));
    else if (dtype == XMOE_F32)
        rbd_merge_kernel<float><<<cap(warp_grid(per)), 256, 0, st>>>(eout_tab, H, desc, gstart, wk.rx, wk.C, c,
                                                                    static_cast<float*>(back_u));
    else if (H % 8 == 0)
        rbd_merge_bf16_kernel<<<cap(warp_grid(per * ((H + 511) / 512))), 256, 0, st>>>(
            eout_tab, H, desc, gstart, wk.rx, wk.C, c, static_cast<__nv_bfloat16*>(back_u));
    else
        rbd_merge_kernel<__nv_bfloat16><<<cap(warp_grid(per)), 256, 0, st>>>(
            eout_tab, H, desc, gstart, wk.rx, wk.C, c, static_cast<__nv_bfloat16*>(back_u));
    XMOE_LAUNCH_CHECK();
}

void launch_rbd_combine(int dtype, const char* const* back_tab, int H, int S, const RbdWork& wk, int c,
                        const double* cw, const void* addend, void* out, cudaStream_t st) {
    const int nt = chunk_t0(c + 1, S, wk.C) - chunk_t0(c, S, wk.C);
    if (nt == 0) return;
    if (dtype == XMOE_F64)
        rbd_combine_kernel<double><<<ceil_div(nt, 8), 256, 0, st>>>(
            back_tab, H, S, wk.gbase, wk.gcount, wk.g, wk.ru, wk.gpos, wk.C, c, wk.dptr, cw,
            static_cast<const double*>(addend), static_cast<double*>(out));
    else if (dtype == XMOE_F32)
        rbd_combine_kernel<float><<<ceil_div(nt, 8), 256, 0, st>>>(
            back_tab, H, S, wk.gbase, wk.gcount, wk.g, wk.ru, wk.gpos, wk.C, c, wk.dptr, cw,
            static_cast<const float*>(addend), static_cast<float*>(out));
    else if (H % 8 == 0 && g_copy_fat > 0) {  // whole-SM blocks of the SM partition
        static bool attr = false;
        if (!attr) {
            XMOE_CUDA(cudaFuncSetAttribute(rbd_combine_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kFatSmemBytes));
            attr = true;
        }
        rbd_combine_bf16_kernel<<<g_copy_fat, 1024, kFatSmemBytes, st>>>(
            back_tab, H, S, wk.gbase, wk.gcount, wk.g, wk.ru, wk.gpos, wk.C, c, wk.dptr, cw,
            static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out));
    } else if (H % 8 == 0)
        rbd_combine_bf16_kernel<<<ceil_div(static_cast<long long>(nt) * ((H + 511) / 512), 8), 256, 0, st>>>(
            back_tab, H, S, wk.gbase, wk.gcount, wk.g, wk.ru, wk.gpos, wk.C, c, wk.dptr, cw,
            static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out));
    else
        rbd_combine_kernel<__nv_bfloat16><<<ceil_div(nt, 8), 256, 0, st>>>(
            back_tab, H, S, wk.gbase, wk.gcount, wk.g, wk.ru, wk.gpos, wk.C, c, wk.dptr, cw,
            static_cast<const __nv_bfloat16*>(addend), static_cast<__nv_bfloat16*>(out));
    XMOE_LAUNCH_CHECK();
}

}  // namespace xmoe
