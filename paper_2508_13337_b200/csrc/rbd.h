// Redundancy-bypassing dispatch: device data structures (see rbd.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace xmoe {

constexpr int kRbdChunk = 256;  // groups per jump-ahead chunk
constexpr int kRbdJumps = 24;   // chunk index < 2^24
constexpr int kRbdPilotFlag = 1 << 16;
constexpr int kRbdMemberMask = 0xFFFF;
constexpr int kRbdOwnerShift = 20;  // member's owner rank (two-tier: may differ from the landing rank)

// One (token, destination rank) group of a source rank, in the reference's
// std::map order (rbd.cpp:35-43).  SoA, indexed by group id.
struct RbdGroups {
    int32_t* token;
    int32_t* dest;
    int32_t* first_slot;  // first member in the token's slot list
    int32_t* n;           // members
    int32_t* pilot;       // packed row of the pilot copy
    int32_t* pos;         // position in the dest-sorted order
};

// Per-copy descriptor riding with the unique rows (24 bytes).
struct RbdDesc {
    int32_t u;         // row of the group in the receiver's unique-row buffer
    int32_t dest_row;  // row of the copy in the receiver's grouped expert input
    double w;          // combine weight of the copy
    int32_t n;         // group size
    int32_t member;    // member index | kRbdPilotFlag | owner rank << kRbdOwnerShift
};
static_assert(sizeof(RbdDesc) == 24, "descriptor layout");

struct RbdWork {
    RbdGroups g;
    int gpn;           // GPUs per node: groups are (token, node); 1 = per-GPU bypass
    int32_t* gcount;   // [S]
    int32_t* gbase;    // [S]
    int32_t* G_dev;    // total groups
    uint64_t* draws;   // [S*k] xoshiro outputs
    int32_t* flags;    // [1] rejection-sampling event seen
    int32_t* dptr;     // [W+1] dest segment starts (dest-sorted)
    int32_t* perm;     // [S*k] dest-sorted position -> group id
    int32_t* nsorted;  // [S*k] group size in sorted order
    int32_t* scan_ws;  // [S*k/2048 + 2] block sums of the multi-block scans
    int32_t* coff;     // [S*k] first descriptor of each sorted group
    void* csr_ws;
    // token chunks (chunk.cu; C = 1 when the forward is not chunked).  The
    // receiver keeps its groups and descriptors in (chunk, source, sender
    // order); a dest segment of the sender is token-ordered, so chunk c of
    // it is the sub-range [gpos[d][c], gpos[d][c+1]).
    int C;
    int32_t* gpos;     // [W, C+1] chunk starts inside each dest segment
    int32_t* gd_own;   // [2, W, C] my groups / copies per (dest, chunk)
    int32_t* ru;       // [W, C] my first group row at receiver d for chunk c
    int32_t* rd;       // [W, C] my first descriptor slot at receiver d for chunk c
    int32_t* cs;       // [W, C] first descriptor (my order) of my (d, c) segment
    int32_t* rx;       // [4, C] receiver: group base, groups, descriptor base, descriptors
    uint64_t state[4];  // Rng(salt_seed(seed, rank, 0)) state
};

uint64_t salt_seed_host(uint64_t seed, uint64_t a, uint64_t b);
void rng_state_from_seed(uint64_t seed, uint64_t out[4]);
void rbd_jump_tables(std::vector<uint64_t>& out);
void gf2_jump_tables(int log2_chunk, int count, std::vector<uint64_t>& out);
// outputs [offset, offset + n) of Rng(seed).uniform(lo, hi) (rng.hpp:24-47)
void launch_rng_uniform(uint64_t seed, unsigned long long offset, long long n, double lo, double hi, double grid,
                        int dtype, void* out, cudaStream_t st);
void launch_rng_uniform_state(const uint64_t s[4], unsigned long long offset, long long n, double lo, double hi,
                              double grid, int dtype, void* out, cudaStream_t st);
void rng_advance(uint64_t s[4], unsigned long long n);

void launch_rbd_groups(const int32_t* slot_pos, const int32_t* expert_ids, int S, int k, int El,
                       const uint64_t state[4], const uint64_t* jumps, RbdWork& wk, cudaStream_t st);
void launch_rbd_sort(int W, long long max_groups, RbdWork& wk, cudaStream_t st);
// per (dest, chunk) group / copy counts of this sender (before the all-gather)
void launch_rbd_chunk_counts(int W, int S, RbdWork& wk, cudaStream_t st);
// offsets from every sender's counts gd_all [W_src, 2, W, C]
void launch_rbd_offsets(const int32_t* gd_all, int W, int me, RbdWork& wk, cudaStream_t st);
// chunk c (tokens [floor(cS/C), floor((c+1)S/C)))
void launch_rbd_pack(const void* x, int row_bytes, const RbdWork& wk, int W, int c, long long max_groups,
                     const int32_t* slot_pos, int k, const int32_t* dest_row, const double* cw,
                     char* const* recv_u_tab, RbdDesc* const* desc_tab, cudaStream_t st, int S = 0,
                     const int32_t* expert_ids = nullptr, int El = 1);
// replicas copy their pilot's row (local) into their owner's grouped input
// (recv_tab: local or NVLink peer); `grouped` is this landing rank's input
// a_idx (gather mode, one GPU per node): record each copy's pilot row for
// the row-gathered GEMM1 instead of copying the row
void launch_rbd_expand(int row_bytes, const RbdDesc* desc, const RbdWork& wk, int c, long long max_desc,
                       void* grouped, char* const* recv_tab, int32_t* gstart, cudaStream_t st,
                       int32_t* a_idx = nullptr);
// each group's members' outputs read from their owners (eout_tab)
void launch_rbd_merge(int dtype, const char* const* eout_tab, int H, const RbdDesc* desc, const int32_t* gstart,
                      const RbdWork& wk, int c, long long max_groups, void* back_u, cudaStream_t st);
void launch_rbd_combine(int dtype, const char* const* back_tab, int H, int S, const RbdWork& wk, int c,
                        const double* cw, const void* addend, void* out, cudaStream_t st);

// ep.cu: pilot mask [B] (and each copy's pilot row) of the drawn groups
void launch_mask_from_groups(const RbdWork& wk, const int32_t* slot_pos, int k, long long max_groups, uint8_t* mask,
                             int32_t* pilot_of, cudaStream_t st);

// rbd.cu: device counters of the byte ledger (layout in rbd.cu); wk == null:
// only out[0] (off-rank (token, destination) groups)
void launch_ledger_counts(const int32_t* slot_pos, int S, int k, const int32_t* expert_ids, int El, int me,
                          const RbdWork* wk, int W, unsigned long long* out, cudaStream_t st);

// pft.cu: stable CSR with the item count on the device (bound n_max).
void launch_stable_csr_dev(const int32_t* keys, const int32_t* n_dev, int n_max, int K, int32_t* ptr,
                           int32_t* perm, void* ws, cudaStream_t st);

}  // namespace xmoe
