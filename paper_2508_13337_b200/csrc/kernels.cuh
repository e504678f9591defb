// Launchers of the xmoe device kernels (one translation unit each).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace xmoe {

constexpr int kRouteTile = 128;  // tokens per gate tile / routing histogram row

// gate.cu
void launch_gate_logits_f64(const double* x, const double* wg, int S, int H, int E,
                            double* logits, cudaStream_t st);
void launch_gate_logits_f32(const float* x, const float* wg, int S, int H, int E, float* logits, cudaStream_t st);
void launch_softmax_topk(const double* logits, int S, int E, int k, int renorm, int32_t* top,
                         double* weights, cudaStream_t st);
// counts (optional): per-128-token-tile expert histograms [ceil(S/128), E]
void launch_softmax_topk_f32(const float* logits, int S, int E, int k, int renorm, int32_t* top,
                             double* weights, cudaStream_t st, int32_t* counts = nullptr);

// pft.cu
size_t bucket_ws_bytes(long long n, int K);
void launch_pft(const int32_t* top, const double* w, int S, int k, int E, int cap,
                int32_t* token_ids, int32_t* expert_ids, double* cw, int32_t* tpe,
                int32_t* slot_pos, int32_t* B_dev, void* ws, cudaStream_t st);
void launch_pft_validate(const int32_t* top, int S, int k, int E, unsigned long long* first_bad,
                         cudaStream_t st);
void launch_stable_csr(const int32_t* keys, int n, int K, int32_t* ptr, int32_t* perm, void* ws,
                       cudaStream_t st);

// permute.cu
void launch_gather_rows(const void* src, long long rows, int row_bytes, const int32_t* ids,
                        long long n, const int32_t* n_dev, void* out, int* err, cudaStream_t st);
void launch_dispatch_dest(const int32_t* tpe_all, int W, int E, int src,
                          const int32_t* expert_ids, const int32_t* B_dev, long long max_rows,
                          int32_t* dest_rank, int32_t* dest_row, cudaStream_t st);
void launch_scatter_rows(const void* x, int row_bytes, const int32_t* token_ids,
                         const int32_t* B_dev, long long max_rows, const int32_t* dest_rank,
                         const int32_t* dest_row, char* const* dest_bufs, cudaStream_t st);
void launch_scatter_tokens(const void* x, int row_bytes, int S, int k, const int32_t* slot_pos,
                           const int32_t* dest_rank, const int32_t* dest_row, const double* cw,
                           char* const* dest_bufs, char* const* src_bufs, unsigned long long* slot_src,
                           float* slot_w, cudaStream_t st);
// out[t] = sum over t's kept copies of w * row(copy) (+ addend[t] + addend2[t]);
// row address = slot_src + src_delta bytes; slot_w == null means weight 1.
void launch_combine_slots(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                          const void* addend, void* out, cudaStream_t st, long long src_delta = 0,
                          const void* addend2 = nullptr);
// routed copies only, fp32 sums to partial [S, H]; ready[t / 128] += 1 per token
void launch_combine_slots_partial(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                                  float* partial, unsigned* ready, cudaStream_t st);
// the same over the warp kernel (fat SM blocks when g_copy_fat > 0): tokens
// t_base.. of a chunk; every (token, 512-column segment) item adds 1 to
// ready[(t_base + t) / 128], so a block is complete at rows x combine_segments(H)
void launch_combine_slots_seg_partial(const unsigned long long* slot_src, const float* slot_w, int k, int H, int S,
                                      float* partial, unsigned* ready, int t_base, cudaStream_t st);
int combine_segments(int H);
void launch_unscatter_rows(int row_bytes, const int32_t* B_dev, long long max_rows,
                           const int32_t* dest_rank, const int32_t* dest_row,
                           const char* const* src_bufs, void* out, cudaStream_t st);

// combine.cu — out[t] = sum over t's copies c (ascending) of w[c] * row(c)
// (+ addend[t]); row(c) = rows[c] or, with a table, tab[drank[c]][drow[c]].
void launch_combine(int dtype, const void* rows, int H, const int32_t* ptr, const int32_t* idx,
                    int k, const double* w, int S, const void* addend, void* out,
                    cudaStream_t st, const char* const* tab = nullptr,
                    const int32_t* drank = nullptr, const int32_t* drow = nullptr);

// gemm_f64.cu
void launch_grouped_gemm_f64(const double* A, long long rows_bound, int K,
                             const int32_t* rows_per_group, int G, const double* B, int N,
                             double* D, int relu, cudaStream_t st);

void launch_grouped_gemm_f32(const float* A, long long rows_bound, int K, const int32_t* rows_per_group, int G,
                             const float* B, int N, float* D, int relu, cudaStream_t st);

// gemm_tc.cu
// mbits_out (ReLU GEMMs, training layers): bit i of word [row][c/32] = (y[row][c] != 0)
void launch_grouped_gemm_bf16(const void* A, long long rows, int K, const int32_t* rows_per_group,
                              int G, const void* B, int N, void* D, int relu, cudaStream_t st,
                              uint32_t* mbits_out = nullptr);
// A rows gathered through a_idx: logical row r (< rows) reads A[a_idx[r]]
// (A has phys_rows rows; TMA gather4)
void launch_grouped_gemm_bf16_gather(const void* A, long long phys_rows, long long rows, int K,
                                     const int32_t* rows_per_group, int G, const void* B, int N, void* D, int relu,
                                     const int32_t* a_idx, cudaStream_t st);
// dgrad with the ReLU mask of the forward: D = (A B) * mask
void launch_grouped_gemm_bf16_mask(const void* A, long long rows, int K, const int32_t* rows_per_group, int G,
                                   const void* B, int N, void* D, const uint32_t* mbits, cudaStream_t st);
void launch_grouped_wgrad_bf16(const void* A, int M, long long Ktot, const int32_t* k_per_group, int G,
                               const void* B, int N, float* D, cudaStream_t st);
void launch_grouped_wgrad_mn(const void* A, int M, const void* B, int N, long long rows,
                             const int32_t* group_rows, int G, void* tail_a, void* tail_b, float* D,
                             cudaStream_t st);
void launch_grouped_wgrad_mn_t(const void* A, int M, const void* B, int N, long long rows,
                               const int32_t* group_rows, int G, void* tail_a, void* tail_b, float* D,
                               cudaStream_t st);
void launch_wgrad_mn_split(const void* A, int M, const void* B, int Nb, long long rows, int splits,
                           int32_t* split_rows, void* tail_a, void* tail_b, float* partial, float* D,
                           cudaStream_t st);
void launch_grouped_gemm_bf16_f32out(const void* A, long long rows, int K,
                                     const int32_t* rows_per_group, int G, const void* B, int N,
                                     float* D, int relu, cudaStream_t st);

// fused gate (gemm_tc.cu): logits GEMM + softmax + top-k from TMEM, per-tile
// expert histograms counts [ceil(S/128), E] (optional), fp32 logits (optional)
bool gate_route_supported(int E, int k, int H);
void launch_gate_route(const void* x, int S, int H, const void* gate_kmajor, int E, int k, int renorm, int32_t* top,
                       double* weights, float* logits, int32_t* counts, cudaStream_t st);
// fused dropless placement (pft.cu) from the gate's tile histograms: the
// packed ERI arrays, tokens_per_expert, slot_pos and B (= S*k)
void launch_route_place(const int32_t* top, const double* weights, const int32_t* counts, int S, int E, int k,
                        int32_t* token_ids, int32_t* expert_ids, double* cw, int32_t* tpe, int32_t* slot_pos,
                        int32_t* B_dev, cudaStream_t st);

// backward.cu
void launch_bwd_owner_prep(const void* dyg, const void* eout, const float* gw, const unsigned long long* gsrc,
                           const int32_t* rpe, int El, int H, long long max_rows, float* const* slotdw_tab,
                           void* dz, int me, cudaStream_t st);
void launch_bwd_scatter_dy(const void* dy, int H, int S, int k, const int32_t* slot_pos, const int32_t* dest_rank,
                           const int32_t* dest_row, const double* cw, int me, void* dz, char* const* eout_tab,
                           char* const* dyg_tab, char* const* dxc_tab, float* const* gw_tab,
                           unsigned long long* const* gsrc_tab, float* slot_dw, unsigned long long* bslot_src,
                           cudaStream_t st);
void launch_pad_offsets(const int32_t* rows, int G, int32_t* kpg, int32_t* koff, int32_t* roff, cudaStream_t st);
void launch_transpose_pad(const void* in, int C, const int32_t* rows, const int32_t* koff, const int32_t* roff,
                          int G, long long ld, void* out, cudaStream_t st);
void launch_gate_bwd(const float* logits, const int32_t* slot_pos, const int32_t* expert_ids, const float* slot_dw,
                     int S, int E, int k, void* dl, cudaStream_t st);

// gemm_tc.cu: SM budget of subsequent 2-CTA GEMM launches on this thread (0 = all)
extern thread_local int g_gemm_sm_limit;
// fused fp32 addend of the next bf16 2-CTA GEMM launches (one group of rows,
// no ReLU): D = bf16(addf[row] + float(bf16(acc))), each 128-row block read
// once ready[block] reaches its row count (published by the partial combine)
extern thread_local const float* g_gemm_addf;
extern thread_local const unsigned* g_gemm_ready;
extern thread_local int g_gemm_ready_mult;  // publications per row the ready counters count (default 1)
bool gemm_2cta_enabled(int N);  // the 2-CTA kernel serves N (XMOE_GEMM, N % 32)
void launch_count_check(const int32_t* rpe, int G, long long rows, int32_t* clamped, int* err, cudaStream_t st);
// grid cap of the row-movement kernels (token scatter, slot combine; 0 =
// their default).  The chunked forward runs them on a few SMs' worth of
// blocks so the NVLink traffic they drive does not stall the GEMM CTAs on
// every SM.
extern thread_local int g_copy_blocks;
// dynamic shared memory the row-movement kernels reserve (unused): large
// enough, it keeps them off SMs that hold a GEMM CTA (SM partition)
extern thread_local int g_copy_smem;
// SM partition of the chunked forward (XMOE_COMM_SMS): when > 0 the row
// pulls and combines that run beside the expert GEMMs launch as this many
// whole-SM blocks (one per SM: 1024 threads + a large shared reservation, or
// the full register file), and the GEMMs take the remaining SMs, so the row
// traffic never shares an SM with a GEMM CTA.
extern thread_local int g_copy_fat;

// Token chunk boundaries of the pipelined forward: chunk c = tokens
// [cS/C, (c+1)S/C); chunk_of(t) inverts chunk_t0.  (Measured on B200, C2
// N=4: a half-size last chunk, or half-size first and last chunks, gave
// 42.7 / 41.6 M tokens/s against 42.4-42.8 M for even chunks, and both cost
// N=2 or C3 — even chunks kept.)
__host__ __device__ __forceinline__ int chunk_t0(int c, long long S, int C) {
    return c >= C ? static_cast<int>(S) : static_cast<int>(c * S / C);
}
__host__ __device__ __forceinline__ int chunk_of(int t, long long S, int C) {
    return static_cast<int>((static_cast<long long>(t + 1) * C - 1) / S);
}
inline long long chunk_max_tokens(long long S, int C) { return (S + C - 1) / C; }
constexpr int kFatSmemBytes = 120 * 1024;  // reservation that keeps one fat block per SM and GEMM CTAs off it

// misc.cu
void launch_recv_counts(const int32_t* tpe_all, int W, int E, int dst, int32_t* rpe,
                        cudaStream_t st);
void launch_fill_i32(int32_t* p, int n, int32_t v, cudaStream_t st);
void launch_adjacent_diff(const int32_t* ptr, int n, int32_t* out, cudaStream_t st);
void launch_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st);
void launch_transpose(int dtype_in, const void* in, int batch, int rows, int cols,
                      int dtype_out, void* out, cudaStream_t st);

// chunk.cu: token-chunked pipeline (layout, counts, cross-GPU epoch flags)
constexpr int kMaxChunks = 8;
void launch_chunk_counts(const int32_t* token_ids, const int32_t* tpe, int E, int S, int C, int32_t* tpe_c,
                         int32_t* pfx_c, int32_t* seg, cudaStream_t st);
void launch_chunk_bases(const int32_t* T, int W, int C, int E, int me, int Rc, int32_t* base, int32_t* rpe_c,
                        cudaStream_t st);
void launch_dispatch_dest_chunked(const int32_t* expert_ids, const int32_t* token_ids, const int32_t* B_dev,
                                  long long max_rows, int S, int C, int E, int El, const int32_t* seg,
                                  const int32_t* pfx_c, const int32_t* base, int32_t* dest_rank,
                                  int32_t* dest_row, cudaStream_t st,
                                  int32_t* const* rsrc_tab = nullptr, int me = 0);
// pull dispatch (chunk.cu): combine addresses per token slot; owner-side row pull
void launch_slot_addrs(const int32_t* slot_pos, long long n, const int32_t* dest_rank, const int32_t* dest_row,
                       const double* cw, char* const* eout_tab, int row_bytes, unsigned long long* slot_src,
                       float* slot_w, cudaStream_t st);
void launch_pull_rows(const int32_t* rsrc, const int32_t* rpe, int El, char* const* xs_tab, int row_bytes,
                      long long max_rows, void* recv, cudaStream_t st);
void launch_forward_begin(int32_t* s_rows, int S, unsigned* epoch, cudaStream_t st);
void launch_flag_signal(unsigned* const* flag_tab, int W, int me, int slot, const unsigned* epoch,
                        cudaStream_t st);
// waits give up after XMOE_PEER_TIMEOUT_S (default 300 s) and record the slot
// in *err (the layer's host-mapped error word) instead of trapping
void launch_flag_wait(const unsigned* flags, int W, int slot, const unsigned* epoch, int* err, cudaStream_t st);
// flag slots per rank: [0, kMaxChunks) chunk dispatch, [kMaxChunks, 2 kMaxChunks)
// chunk combine, then the count exchange, the unchunked forward's barriers
// and the backward's two barriers (same epoch as the forward they follow)
constexpr int kSlotCounts = 2 * kMaxChunks;
constexpr int kSlotBar = 2 * kMaxChunks + 1;     // + 0..3
constexpr int kSlotBwdBar = 2 * kMaxChunks + 5;  // + 0..1
constexpr int kSlotQuiesce = 2 * kMaxChunks + 7;  // layer teardown
constexpr int kFlagSlots = 2 * kMaxChunks + 8;
struct CountSeg {
    const int32_t* src;  // my row
    int row;             // ints per rank row
    int off;             // offset of the [W, row] block in the count area
    int32_t* local;      // [W, row] gathered copy
};
struct CountSegs {
    CountSeg s[4];
    int n;
};
void launch_counts_exchange(const CountSegs& segs, int32_t* const* area_tab, int area_ints, int me, int W,
                            unsigned* const* flag_tab, const unsigned* my_flags, int slot, const unsigned* epoch,
                            int* err, cudaStream_t st);
void launch_flag_barrier(unsigned* const* flag_tab, const unsigned* my_flags, int W, int me, int slot,
                         const unsigned* epoch, int* err, cudaStream_t st);

}  // namespace xmoe
