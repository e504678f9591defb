// Padding-free token buffer construction — B200 restatement of
// moesim::pft_construct (/root/reference/proj/src/pft.cpp:12-60).
//
// The reference buckets routing positions f = t*k + j by expert in ascending
// f, keeps at most `cap` per expert by (weight desc, f asc) and emits the
// survivors expert-major, ascending f.  On the GPU that is a stable counting
// sort with a per-expert top-cap selection:
//
//   K1 bucket_count   warp-aggregated histogram per 512-entry chunk
//                     (__match_any_sync groups lanes hitting one expert)
//   K2 bucket_scan    one CTA: column scan over chunks, capacity clamp,
//                     exclusive scans over experts (raw and kept layouts)
//   K3 bucket_place   every warp re-walks its chunk in order; positions are
//                     running count + rank among matching lanes, so the
//                     order is stable (= ascending f within an expert)
//   K4 capacity_select  one CTA per over-full expert: 96-bit radix select of
//                     the cap-th key (weight bits, ~f), order-preserving
//                     compaction (only launched work when some expert overflows)
//   K5 pft_finalize   kept copies -> token_ids / expert_ids / weights
//   K6 slot_sort      per token, its kept rows ascending (for the combine)
#include "common.cuh"
#include "kernels.cuh"
#include "rbd.h"

namespace xmoe {

constexpr int kChunk = 512;   // entries per warp chunk (16 warp steps)
constexpr int kWarps = 8;     // warps per CTA in K1/K3

struct BucketWs {
    int32_t* counts;     // [nchunks, K] per-chunk histogram, then running offsets
    int32_t* raw_cnt;    // [K]
    int32_t* raw_base;   // [K+1]
    int32_t* kept_base;  // [K+1]
    int32_t* sorted_f;   // [n]  dropless stable order (raw layout)
    int32_t* newidx;     // [n]  index within expert after capacity (-1 dropped)
    int32_t* fpos;       // [n]  flat position -> final packed row (-1 dropped)
    int32_t* flags;      // [4]  0: any overflow, 1: error code, 2: error detail
};

// ---------------------------------------------------------------- validation
// Reference order of checks (pft.cpp:23-31): row-major over (t, a); the first
// offending entry decides IndexError (out of range) vs ValidationError
// (duplicate within a row).  We record the smallest offending flat index and
// its kind with one atomicMin on (f << 1 | kind).
__global__ void pft_validate_kernel(const int32_t* __restrict__ top, int S, int k, int E,
                                    unsigned long long* __restrict__ first_bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int32_t* r = top + static_cast<size_t>(t) * k;
    for (int a = 0; a < k; ++a) {
        const int e = r[a];
        int kind = -1;
        if (e < 0 || e >= E) kind = 0;  // IndexError
        else
            for (int b = 0; b < a; ++b)
                if (r[b] == e) kind = 1;  // ValidationError
        if (kind >= 0) {
            const unsigned long long key =
                (static_cast<unsigned long long>(static_cast<size_t>(t) * k + a) << 1) | kind;
            atomicMin(first_bad, key);
            return;
        }
    }
}

// ---------------------------------------------------------------- K1
template <bool kSmem>
__global__ void __launch_bounds__(32 * kWarps) bucket_count_kernel(
    const int32_t* __restrict__ keys, int n_host, const int32_t* __restrict__ n_dev, int K,
    int32_t* __restrict__ counts) {
    extern __shared__ int32_t hist[];  // [kWarps][K] when kSmem
    const int n = n_dev ? *n_dev : n_host;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chunk = blockIdx.x * kWarps + warp;
    int32_t* h = kSmem ? hist + warp * K : counts + static_cast<size_t>(chunk) * K;
    if (kSmem)
        for (int i = lane; i < K; i += 32) h[i] = 0;
    __syncwarp();
    const int f0 = chunk * kChunk;
    for (int s = 0; s < kChunk; s += 32) {
        const int f = f0 + s + lane;
        const bool valid = f < n;
        const int key = valid ? keys[f] : -1;
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        if (!valid) continue;
        const unsigned peers = __match_any_sync(active, key);
        if ((peers & lanemask_lt()) == 0) {  // lowest lane of the group adds the group
            if (kSmem) h[key] += __popc(peers);
            else atomicAdd(h + key, __popc(peers));
        }
        __syncwarp(active);
    }
    __syncwarp();
    if (kSmem && f0 < n)
        for (int i = lane; i < K; i += 32) counts[static_cast<size_t>(chunk) * K + i] = h[i];
    else if (kSmem)
        for (int i = lane; i < K; i += 32) counts[static_cast<size_t>(chunk) * K + i] = 0;
}

// ---------------------------------------------------------------- K2
// Single CTA.  Phase 1, one warp per key: warp-parallel exclusive scan of the
// key's per-chunk counts (in place), raw total and capacity-clamped total.
// Phase 2: block-wide exclusive scans over keys of both totals.
// raw_base/kept_base get K+1 entries (last = totals).
__global__ void __launch_bounds__(1024) bucket_scan_kernel(int nchunks, int K, int cap,
                                                           int32_t* __restrict__ counts,
                                                           int32_t* __restrict__ raw_cnt,
                                                           int32_t* __restrict__ raw_base,
                                                           int32_t* __restrict__ kept_base,
                                                           int32_t* __restrict__ kept_cnt,
                                                           int32_t* __restrict__ flags,
                                                           int32_t* __restrict__ total_out) {
    __shared__ int32_t s_raw[1024], s_kept[1024];
    __shared__ int32_t carry_raw, carry_kept;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int any_over = 0;
    for (int key = warp; key < K; key += 32) {
        int running = 0;
        for (int c0 = 0; c0 < nchunks; c0 += 32) {
            const int c = c0 + lane;
            const int v = c < nchunks ? counts[static_cast<size_t>(c) * K + key] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (c < nchunks) counts[static_cast<size_t>(c) * K + key] = running + incl - v;
            running += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            raw_cnt[key] = running;
            if (kept_cnt) kept_cnt[key] = min(running, cap);
            if (running > cap) any_over = 1;
        }
    }
    if (threadIdx.x == 0) {
        carry_raw = 0;
        carry_kept = 0;
    }
    __syncthreads();
    for (int k0 = 0; k0 < K; k0 += 1024) {
        const int key = k0 + threadIdx.x;
        const int tot = key < K ? raw_cnt[key] : 0;
        const int kept = key < K ? min(tot, cap) : 0;
        s_raw[threadIdx.x] = tot;
        s_kept[threadIdx.x] = kept;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scans
            const int a = threadIdx.x >= o ? s_raw[threadIdx.x - o] : 0;
            const int b = threadIdx.x >= o ? s_kept[threadIdx.x - o] : 0;
            __syncthreads();
            s_raw[threadIdx.x] += a;
            s_kept[threadIdx.x] += b;
            __syncthreads();
        }
        if (key < K) {
            raw_base[key] = carry_raw + s_raw[threadIdx.x] - tot;
            kept_base[key] = carry_kept + s_kept[threadIdx.x] - kept;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry_raw += s_raw[1023];
            carry_kept += s_kept[1023];
        }
        __syncthreads();
    }
    any_over = __syncthreads_or(any_over);
    if (threadIdx.x == 0) {
        raw_base[K] = carry_raw;
        kept_base[K] = carry_kept;
        flags[0] = any_over;
        if (total_out) *total_out = carry_kept;
    }
}

// ---------------------------------------------------------------- K3
// counts[c][key] holds the exclusive per-chunk offset within the key; the
// final raw position is raw_base[key] + that + running rank.
template <bool kSmem>
__global__ void __launch_bounds__(32 * kWarps) bucket_place_kernel(
    const int32_t* __restrict__ keys, int n_host, const int32_t* __restrict__ n_dev, int K,
    int32_t* __restrict__ counts, const int32_t* __restrict__ raw_base,
    int32_t* __restrict__ sorted_f) {
    extern __shared__ int32_t run[];
    const int n = n_dev ? *n_dev : n_host;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chunk = blockIdx.x * kWarps + warp;
    const int f0 = chunk * kChunk;
    if (f0 >= n) return;
    int32_t* r = kSmem ? run + warp * K : counts + static_cast<size_t>(chunk) * K;
    if (kSmem)
        for (int i = lane; i < K; i += 32) r[i] = counts[static_cast<size_t>(chunk) * K + i] + raw_base[i];
    __syncwarp();
    for (int s = 0; s < kChunk; s += 32) {
        if (f0 + s >= n) break;  // warp-uniform
        const int f = f0 + s + lane;
        const bool valid = f < n;
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int key = keys[f];
            const unsigned peers = __match_any_sync(active, key);
            const int rank = __popc(peers & lanemask_lt());
            const int base = kSmem ? r[key] : r[key] + raw_base[key];
            sorted_f[base + rank] = f;
            __syncwarp(active);
            if (rank == __popc(peers) - 1) r[key] += __popc(peers);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- K4
// Doubles mapped to unsigned keys with the same total order (-0.0 == +0.0,
// as the reference's `!=`/`>` comparisons treat them, pft.cpp:44-46).
__device__ __forceinline__ unsigned long long order_key(double v) {
    if (v == 0.0) v = 0.0;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// One CTA per key.  Keys with raw count <= cap keep everything (identity
// newidx).  Over-full keys: radix select (8-bit digits, most significant
// first) of the cap-th largest 96-bit key  (weight bits << 32 | ~f)  —
// positive doubles order like their bit patterns, ~f makes the earlier
// routing position win ties (pft.cpp:42-47) — then an order-preserving
// compaction of the survivors (pft.cpp:49-50 re-sorts by f).
__global__ void __launch_bounds__(1024) capacity_select_kernel(
    const int32_t* __restrict__ sorted_f, const double* __restrict__ w,
    const int32_t* __restrict__ raw_cnt, const int32_t* __restrict__ raw_base, int cap,
    const int32_t* __restrict__ flags, int32_t* __restrict__ newidx) {
    const int key = blockIdx.x;
    const int n = raw_cnt[key];
    const int base = raw_base[key];
    if (!flags[0]) return;  // no expert overflowed: K5 uses the raw layout
    if (n <= cap) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) newidx[base + i] = i;
        return;
    }
    __shared__ int hist[256];
    __shared__ unsigned long long s_prefix_hi;
    __shared__ unsigned s_prefix_lo;
    __shared__ int s_remaining;
    __shared__ int s_warp_sums[32];
    if (threadIdx.x == 0) {
        s_prefix_hi = 0;
        s_prefix_lo = 0;
        s_remaining = cap;
    }
    __syncthreads();
    // 12 digits: 8 from the weight bits (hi), 4 from ~f (lo).
    for (int d = 0; d < 12; ++d) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const int shift_hi = 56 - 8 * d;       // d < 8
        const int shift_lo = 24 - 8 * (d - 8);  // d >= 8
        const unsigned long long ph = s_prefix_hi;
        const unsigned pl = s_prefix_lo;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int f = sorted_f[base + i];
            const unsigned long long hi = order_key(w[f]);
            const unsigned lo = ~static_cast<unsigned>(f);
            bool match;
            int digit;
            if (d < 8) {
                match = (d == 0) || ((hi >> (shift_hi + 8)) == (ph >> (shift_hi + 8)));
                digit = static_cast<int>((hi >> shift_hi) & 0xff);
            } else {
                match = hi == ph && (d == 8 || (lo >> (shift_lo + 8)) == (pl >> (shift_lo + 8)));
                digit = static_cast<int>((lo >> shift_lo) & 0xff);
            }
            if (match) atomicAdd(&hist[digit], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // walk digits from the top; find where the remaining count falls
            int rem = s_remaining;
            int dig = 255;
            for (; dig > 0; --dig) {
                if (hist[dig] >= rem) break;
                rem -= hist[dig];
            }
            s_remaining = rem;
            if (d < 8) s_prefix_hi |= static_cast<unsigned long long>(dig) << shift_hi;
            else s_prefix_lo |= static_cast<unsigned>(dig) << shift_lo;
        }
        __syncthreads();
    }
    // Threshold key T = (s_prefix_hi, s_prefix_lo) is the cap-th largest; keys
    // are unique (f unique) so exactly cap members satisfy key >= T.
    const unsigned long long th = s_prefix_hi;
    const unsigned tl = s_prefix_lo;
    // order-preserving compaction in tiles of blockDim
    int carry = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        int keep = 0;
        if (i < n) {
            const int f = sorted_f[base + i];
            const unsigned long long hi = order_key(w[f]);
            const unsigned lo = ~static_cast<unsigned>(f);
            keep = (hi > th) || (hi == th && lo >= tl);
        }
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_warp_sums[wid] = __popc(b);
        __syncthreads();
        int before = 0;
        for (int q = 0; q < wid; ++q) before += s_warp_sums[q];
        int tile_total = 0;
        for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) tile_total += s_warp_sums[q];
        if (i < n) newidx[base + i] = keep ? carry + before + __popc(b & lanemask_lt()) : -1;
        carry += tile_total;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- K5
__global__ void pft_finalize_kernel(const int32_t* __restrict__ sorted_f,
                                    const double* __restrict__ w, int n, int k, int E,
                                    const int32_t* __restrict__ raw_base,
                                    const int32_t* __restrict__ kept_base,
                                    const int32_t* __restrict__ newidx,
                                    const int32_t* __restrict__ flags,
                                    int32_t* __restrict__ token_ids,
                                    int32_t* __restrict__ expert_ids, double* __restrict__ cw,
                                    int32_t* __restrict__ fpos) {
    extern __shared__ int32_t s_base[];  // raw_base[0..E]
    for (int i = threadIdx.x; i <= E; i += blockDim.x) s_base[i] = raw_base[i];
    __syncthreads();
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    // expert of raw slot p: last e with raw_base[e] <= p
    int lo = 0, hi = E - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_base[mid] <= p) lo = mid;
        else hi = mid - 1;
    }
    const int e = lo;
    const int f = sorted_f[p];
    const int idx = flags[0] ? newidx[p] : p - s_base[e];
    if (idx < 0) {
        if (fpos) fpos[f] = -1;
        return;
    }
    const int pos = kept_base[e] + idx;
    token_ids[pos] = f / k;
    expert_ids[pos] = e;
    cw[pos] = w[f];
    if (fpos) fpos[f] = pos;
}

// ---------------------------------------------------------------- K6
__global__ void slot_sort_kernel(const int32_t* __restrict__ fpos, int S, int k,
                                 int32_t* __restrict__ slot_pos) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    int v[16];
    int m = 0;
    const int32_t* r = fpos + static_cast<size_t>(t) * k;
    int32_t* o = slot_pos + static_cast<size_t>(t) * k;
    if (k <= 16) {
        for (int j = 0; j < k; ++j) {
            const int x = r[j];
            if (x < 0) continue;
            int q = m++;
            while (q > 0 && v[q - 1] > x) {
                v[q] = v[q - 1];
                --q;
            }
            v[q] = x;
        }
        for (int j = 0; j < k; ++j) o[j] = j < m ? v[j] : -1;
    } else {
        // general k: selection of ascending values straight into the output
        int last = -1;
        for (int j = 0; j < k; ++j) {
            int best = 0x7fffffff;
            for (int q = 0; q < k; ++q)
                if (r[q] > last && r[q] < best) best = r[q];
            o[j] = best == 0x7fffffff ? -1 : best;
            if (best != 0x7fffffff) last = best;
        }
    }
}

// ---------------------------------------------------------------- fused dropless placement
// pft_construct (pft.cpp:12-60) when no bucket can overflow (cap >= S: every
// expert holds at most one copy per token), in one launch from the gate's
// per-tile expert histograms (gemm_tc.cu gate_route_kernel).  Block b owns
// tokens [128 b, 128 b + 128):
//   base[e] = (copies of experts < e) + (copies of e in tiles < b)
//   rank    = tokens t' < t of this tile routed to e: a 128-bit token mask per
//             expert (atomicOr, order-free) and a popcount below t
// so copy (t, e) lands at packed row base[e] + rank — experts ascending,
// tokens ascending inside an expert: the reference's order, bit for bit.
// Each token's kept rows are then written ascending (slot_pos).
__global__ void __launch_bounds__(256) route_place_kernel(const int32_t* __restrict__ top,
                                                          const double* __restrict__ w,
                                                          const int32_t* __restrict__ counts, int nt, int S, int E,
                                                          int k, int32_t* __restrict__ token_ids,
                                                          int32_t* __restrict__ expert_ids, double* __restrict__ cw,
                                                          int32_t* __restrict__ tpe, int32_t* __restrict__ slot_pos,
                                                          int32_t* __restrict__ B_dev) {
    __shared__ int32_t tot[256], base[256];
    __shared__ uint32_t mask[256][4];
    const int b = blockIdx.x, tid = threadIdx.x;
    for (int e = tid; e < E; e += blockDim.x) {
        int all = 0, before = 0;
        for (int q = 0; q < nt; ++q) {
            const int c = counts[static_cast<size_t>(q) * E + e];
            all += c;
            if (q < b) before += c;
        }
        tot[e] = all;
        base[e] = before;
#pragma unroll
        for (int q = 0; q < 4; ++q) mask[e][q] = 0u;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of tot over experts (E <= 256: 8 per lane)
        int v[8], run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid * 8 + q;
            v[q] = e < E ? tot[e] : 0;
            run += v[q];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        int ex = incl - run;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid * 8 + q;
            if (e < E) {
                base[e] += ex;
                if (b == 0) tpe[e] = v[q];
            }
            ex += v[q];
        }
        if (b == 0 && tid == 0) *B_dev = S * k;
    }
    const int t = tid, tok = b * kRouteTile + t;
    const bool ok = t < kRouteTile && tok < S;
    if (ok)
        for (int j = 0; j < k; ++j) {
            const int e = top[static_cast<size_t>(tok) * k + j];
            atomicOr(&mask[e][t >> 5], 1u << (t & 31));
        }
    __syncthreads();
    if (!ok) return;
    int pos[32];
    for (int j = 0; j < k; ++j) {
        const int e = top[static_cast<size_t>(tok) * k + j];
        int r = __popc(mask[e][t >> 5] & ((1u << (t & 31)) - 1u));
        for (int q = 0; q < (t >> 5); ++q) r += __popc(mask[e][q]);
        const int p = base[e] + r;
        token_ids[p] = tok;
        expert_ids[p] = e;
        cw[p] = w[static_cast<size_t>(tok) * k + j];
        int q = j;  // insertion: kept rows ascending (= experts ascending)
        while (q > 0 && pos[q - 1] > p) {
            pos[q] = pos[q - 1];
            --q;
        }
        pos[q] = p;
    }
    for (int j = 0; j < k; ++j) slot_pos[static_cast<size_t>(tok) * k + j] = pos[j];
}

void launch_route_place(const int32_t* top, const double* weights, const int32_t* counts, int S, int E, int k,
                        int32_t* token_ids, int32_t* expert_ids, double* cw, int32_t* tpe, int32_t* slot_pos,
                        int32_t* B_dev, cudaStream_t st) {
    require(E <= 256 && k <= 32, XMOE_ERR_VALIDATION, "fused placement: num_experts <= 256, top_k <= 32");
    if (S == 0) {
        XMOE_CUDA(cudaMemsetAsync(tpe, 0, sizeof(int32_t) * E, st));
        XMOE_CUDA(cudaMemsetAsync(B_dev, 0, sizeof(int32_t), st));
        return;
    }
    const int nt = (S + kRouteTile - 1) / kRouteTile;
    route_place_kernel<<<nt, 256, 0, st>>>(top, weights, counts, nt, S, E, k, token_ids, expert_ids, cw, tpe,
                                           slot_pos, B_dev);
    XMOE_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- host side
size_t bucket_ws_bytes(long long n, int K) {
    const long long nchunks = (n + kChunk - 1) / kChunk + 1;
    size_t b = 0;
    b += sizeof(int32_t) * nchunks * K;  // counts
    b += sizeof(int32_t) * (3 * (K + 1) + 8);
    b += sizeof(int32_t) * 3 * (n + 1);
    return b + 1024;
}

static BucketWs carve(void* ws, long long n, int K) {
    const long long nchunks = (n + kChunk - 1) / kChunk + 1;
    auto* p = static_cast<int32_t*>(ws);
    BucketWs b;
    b.counts = p;
    p += nchunks * K;
    b.raw_cnt = p;
    p += K + 1;
    b.raw_base = p;
    p += K + 1;
    b.kept_base = p;
    p += K + 1;
    b.flags = p;
    p += 8;
    b.sorted_f = p;
    p += n + 1;
    b.newidx = p;
    p += n + 1;
    b.fpos = p;
    return b;
}

// Stable counting sort of keys[0..n) into K buckets with a per-bucket cap.
// Outputs raw_base/kept_base and, per K5, the packed arrays.
void launch_pft(const int32_t* top, const double* w, int S, int k, int E, int cap,
                int32_t* token_ids, int32_t* expert_ids, double* cw, int32_t* tpe,
                int32_t* slot_pos, int32_t* B_dev, void* ws, cudaStream_t st) {
    const long long n = static_cast<long long>(S) * k;
    BucketWs b = carve(ws, n, E);
    const int nchunks = ceil_div(n, kChunk);
    const int nblocks = ceil_div(nchunks, kWarps);
    XMOE_CUDA(cudaMemsetAsync(b.flags, 0, 8 * sizeof(int32_t), st));
    if (n == 0) {
        XMOE_CUDA(cudaMemsetAsync(tpe, 0, sizeof(int32_t) * E, st));
        XMOE_CUDA(cudaMemsetAsync(B_dev, 0, sizeof(int32_t), st));
        return;
    }
    const bool smem = E <= 1536;
    const size_t smem_bytes = smem ? sizeof(int32_t) * kWarps * E : 0;
    if (!smem) XMOE_CUDA(cudaMemsetAsync(b.counts, 0, sizeof(int32_t) * nblocks * kWarps * E, st));
    if (smem) {
        bucket_count_kernel<true><<<nblocks, 32 * kWarps, smem_bytes, st>>>(top, n, nullptr, E, b.counts);
    } else {
        bucket_count_kernel<false><<<nblocks, 32 * kWarps, 0, st>>>(top, n, nullptr, E, b.counts);
    }
    XMOE_LAUNCH_CHECK();
    bucket_scan_kernel<<<1, 1024, 0, st>>>(nblocks * kWarps, E, cap, b.counts, b.raw_cnt,
                                           b.raw_base, b.kept_base, tpe, b.flags, B_dev);
    XMOE_LAUNCH_CHECK();
    if (smem) {
        bucket_place_kernel<true><<<nblocks, 32 * kWarps, smem_bytes, st>>>(
            top, n, nullptr, E, b.counts, b.raw_base, b.sorted_f);
    } else {
        bucket_place_kernel<false><<<nblocks, 32 * kWarps, 0, st>>>(top, n, nullptr, E, b.counts,
                                                                      b.raw_base, b.sorted_f);
    }
    XMOE_LAUNCH_CHECK();
    capacity_select_kernel<<<E, 1024, 0, st>>>(b.sorted_f, w, b.raw_cnt, b.raw_base, cap,
                                               b.flags, b.newidx);
    XMOE_LAUNCH_CHECK();
    pft_finalize_kernel<<<ceil_div(n, 256), 256, sizeof(int32_t) * (E + 1), st>>>(
        b.sorted_f, w, n, k, E, b.raw_base, b.kept_base, b.newidx, b.flags, token_ids,
        expert_ids, cw, slot_pos ? b.fpos : nullptr);
    XMOE_LAUNCH_CHECK();
    if (slot_pos) {
        slot_sort_kernel<<<ceil_div(S, 256), 256, 0, st>>>(b.fpos, S, k, slot_pos);
        XMOE_LAUNCH_CHECK();
    }
}

void launch_pft_validate(const int32_t* top, int S, int k, int E, unsigned long long* first_bad,
                         cudaStream_t st) {
    if (S == 0) return;
    pft_validate_kernel<<<ceil_div(S, 256), 256, 0, st>>>(top, S, k, E, first_bad);
    XMOE_LAUNCH_CHECK();
}

// Stable CSR of arbitrary keys (token ids for scatter_combine, destination
// ranks for RBD groups): perm[pos] = i with positions grouped by key
// ascending and i ascending within a key.  The item count is n_host, or
// *n_dev (bounded by n_host) when n_dev is given.
void launch_stable_csr_dev(const int32_t* keys, const int32_t* n_dev, int n, int K, int32_t* ptr,
                           int32_t* perm, void* ws, cudaStream_t st) {
    BucketWs b = carve(ws, n, K);
    if (n == 0) {
        XMOE_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (K + 1), st));
        return;
    }
    const int nchunks = ceil_div(n, kChunk);
    const int nblocks = ceil_div(nchunks, kWarps);
    const bool smem = K <= 1536;
    const size_t smem_bytes = smem ? sizeof(int32_t) * kWarps * K : 0;
    if (!smem) XMOE_CUDA(cudaMemsetAsync(b.counts, 0, sizeof(int32_t) * nblocks * kWarps * K, st));
    if (smem) bucket_count_kernel<true><<<nblocks, 32 * kWarps, smem_bytes, st>>>(keys, n, n_dev, K, b.counts);
    else bucket_count_kernel<false><<<nblocks, 32 * kWarps, 0, st>>>(keys, n, n_dev, K, b.counts);
    XMOE_LAUNCH_CHECK();
    bucket_scan_kernel<<<1, 1024, 0, st>>>(nblocks * kWarps, K, 0x7fffffff, b.counts, b.raw_cnt,
                                           ptr, b.kept_base, nullptr, b.flags, nullptr);
    XMOE_LAUNCH_CHECK();
    if (smem)
        bucket_place_kernel<true><<<nblocks, 32 * kWarps, smem_bytes, st>>>(keys, n, n_dev, K, b.counts, ptr, perm);
    else
        bucket_place_kernel<false><<<nblocks, 32 * kWarps, 0, st>>>(keys, n, n_dev, K, b.counts, ptr, perm);
    XMOE_LAUNCH_CHECK();
}

void launch_stable_csr(const int32_t* keys, int n, int K, int32_t* ptr, int32_t* perm, void* ws,
                       cudaStream_t st) {
    launch_stable_csr_dev(keys, nullptr, n, K, ptr, perm, ws, st);
}

}  // namespace xmoe
