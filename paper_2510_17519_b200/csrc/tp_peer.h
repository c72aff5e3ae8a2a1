// Tensor-parallel exchange over NVLink peer memory (replaces the NCCL all-reduce of the
// N x H fp32 partial that ends each row-parallel branch of the Megatron head/column split).
//
// Every TP rank owns one peer arena, mapped into all other ranks with CUDA IPC:
//   [flags: u64 [2 phases][kMaxTp sources]] [mailbox: P slots x rpr rows x H] [result: P*rpr rows x H]
// (payload fp32, or bf16 with MGV_TP_PAYLOAD=bf16 in bf16 mode: SURVEY 8(e)'s bytes)
// with rpr = ceil(N / P) rows owned per rank.  One exchange (epoch e, monotonically increasing):
//   1. the row-parallel GEMM's epilogue (EpiF32Peer) writes rows of its partial owned by rank o into
//      slot `self` of o's mailbox (the reduce-scatter transfer, overlapped with the GEMM tile by tile);
//   2. tp_signal: after a system-scope fence, flag[0][self] = e in every owner's arena;
//   3. tp_reduce_gather (owner o): wait for flag[0][*] >= e, sum the P slots in rank order (deterministic,
//      no atomics; bit-identical to accumulating the partials in rank order), write the summed rows into
//      every rank's result region (the all-gather);
//   4. tp_signal flag[1][self] = e everywhere; tp_wait: flag[1][*] >= e, after which the full sum is in the
//      local result region.
// Slot reuse is safe: a rank writes epoch e+1 into a mailbox only after its own wait of epoch e, which
// follows every owner's reduce of epoch e.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "epilogue.cuh"

namespace mgv {

constexpr int64_t kTpFlagBytes = 256;  // 2 x kMaxTp u64 flags, padded

struct TpFlagPtrs {
    unsigned long long* f[kMaxTp];
};
struct TpDstPtrs {
    void* p[kMaxTp];
};

void tp_signal(const TpFlagPtrs& f, int n, uint64_t epoch, cudaStream_t s);
// bf16: mailbox slots and result rows are bf16 (the partials rounded once by the GEMM epilogue; the sum is fp32,
// rounded to bf16 for the all-gather) -- half the bytes over NVLink.  H % 8 == 0.
void tp_reduce_gather(const void* mbox, bool bf16, int P, int64_t rpr, int64_t rows, int64_t H, const TpDstPtrs& dst,
                      int ndst, const unsigned long long* flags, uint64_t epoch, cudaStream_t s);
// the local result region (bf16) -> the fp32 sum the block's consumers read
void tp_bf16_to_f32(const void* in, int64_t n, float* out, cudaStream_t s);
void tp_wait(const unsigned long long* flags, int P, uint64_t epoch, cudaStream_t s);

}  // namespace mgv
