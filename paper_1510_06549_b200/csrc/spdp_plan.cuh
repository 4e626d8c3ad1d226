// spdp_plan.cuh — device-side load planning (spdp_load_corpus).
//
// The wave plan of DESIGN.md §6 (tokens sorted stably by (wave, w, i), wave =
// in-document position mod W — the paper's word-order rearrangement
// P:2289-2299 made deterministic, reading c13; chunks of <= chunk_tokens
// tokens of one (w, i) segment, longest first within a wave; the distinct
// segments of each wave; the doc -> sorted-position CSR) is built with CUB
// radix sorts (stable LSD: ties keep canonical order), run-length encoding and
// scans on the device, so loading costs milliseconds instead of host sorting.
// The plan is a pure function of the corpus; it fixes work units and memory
// order only, never a sampling decision (results do not depend on it).
#pragma once
#include <cub/cub.cuh>

#include "spdp_device.cuh"

namespace spdp {

// range checks, one group per document, document lengths
__global__ void validate_tokens_kernel(const int32_t* __restrict__ group, const int32_t* __restrict__ doc,
                                       const int32_t* __restrict__ word, uint32_t n, int I, int V, int D,
                                       int32_t* __restrict__ docgroup, int32_t* __restrict__ doclen,
                                       unsigned long long* __restrict__ err) {
    // the lanes of a warp that hold the same document (consecutive tokens usually do) act through one
    // leader: one CAS of the document's group and one length add per document and warp, instead of two
    // same-address atomics per token
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t p0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); p0 < n; p0 += stride) {   // warp-uniform
        const uint32_t p = p0 + (threadIdx.x & 31u);
        int32_t g = 0, d = 0, w = 0;
        bool ok = false;
        if (p < n) {
            g = group[p]; d = doc[p]; w = word[p];
            ok = !(g < 0 || g >= I || d < 0 || d >= D || w < 0 || w >= V);
            if (!ok) atomicMin(err, (unsigned long long)p);
        }
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        if (!ok) continue;
        const unsigned peers = __match_any_sync(okm, d);
        const int leader = __ffs(peers) - 1;
        const int32_t gl = __shfl_sync(okm, g, leader);
        if (g != gl) atomicMin(err + 1, (unsigned long long)p);          // the document spans groups in this warp
        if ((int)(threadIdx.x & 31u) == leader) {
            const int32_t old = atomicCAS(docgroup + d, -1, g);
            if (old != -1 && old != g) atomicMin(err + 1, (unsigned long long)p);
            atomicAdd(doclen + d, __popc(peers));
        }
    }
}

// count(i, w) histogram (M_max = its maximum)
__global__ void cell_count_kernel(const int32_t* __restrict__ group, const int32_t* __restrict__ word, uint32_t n,
                                  int V, int32_t* __restrict__ cnt) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        atomicAdd(cnt + (size_t)group[p] * V + word[p], 1);
}

__global__ void iota_kernel(uint32_t* __restrict__ x, uint32_t n) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) x[p] = p;
}

// in-document position l = rank of the token among its document's tokens in canonical order
__global__ void positions_kernel(const uint32_t* __restrict__ by_doc, const int32_t* __restrict__ doc,
                                 const uint32_t* __restrict__ doc_start, uint32_t n, int32_t* __restrict__ pos) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t p = by_doc[j];
        pos[p] = (int32_t)(j - doc_start[doc[p]]);
    }
}

// this rank's tokens (canonical order is kept by the flagged selection)
__global__ void local_flags_kernel(const int32_t* __restrict__ doc, const int32_t* __restrict__ shard, int rank,
                                   uint32_t n, uint8_t* __restrict__ flag) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        flag[p] = shard[doc[p]] == rank;
}

// sort key of a local token: (wave, segment = w * I + i)
__global__ void plan_keys_kernel(const uint32_t* __restrict__ local, uint32_t nloc, const int32_t* __restrict__ group,
                                 const int32_t* __restrict__ word, const int32_t* __restrict__ pos, int I, int W,
                                 uint64_t S, uint64_t* __restrict__ key) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nloc; q += gridDim.x * blockDim.x) {
        const uint32_t p = local[q];
        const uint64_t wave = (W == 1) ? 0u : (uint64_t)(pos[p] % W);   // (W = 1: positions not computed)
        key[q] = wave * S + (uint64_t)word[p] * (uint64_t)I + (uint64_t)group[p];
    }
}

// begin[v] = first index j with f(j) >= v for a non-decreasing f over [0, n); begin[nv] = n
template <typename F>
__global__ void bounds_kernel(F f, uint32_t n, uint32_t nv, uint32_t* __restrict__ begin) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += gridDim.x * blockDim.x) {
        const uint64_t prev = j > 0 ? f(j - 1) + 1 : 0;
        const uint64_t cur = j < n ? f(j) : nv;
        for (uint64_t v = prev; v <= cur && v <= nv; ++v) begin[v] = j;
    }
}
struct WaveOfKey {
    const uint64_t* key;
    uint64_t S;
    __device__ uint64_t operator()(uint32_t j) const { return key[j] / S; }
};
struct WaveOfChunkKey {
    const uint64_t* key;
    uint64_t span;
    __device__ uint64_t operator()(uint32_t j) const { return key[j] / span; }
};

__global__ void chunk_count_kernel(const uint32_t* __restrict__ run_len, uint32_t R, uint32_t chunk,
                                   uint32_t* __restrict__ nch) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x)
        nch[r] = (run_len[r] + chunk - 1) / chunk;
}

// chunks of each run (segment of a wave), in segment order; sort key (wave, longest first)
__global__ void chunk_emit_kernel(const uint64_t* __restrict__ run_key, const uint32_t* __restrict__ run_len,
                                  const uint32_t* __restrict__ run_off, const uint32_t* __restrict__ chunk_off,
                                  uint32_t R, uint32_t chunk, uint64_t S, const uint32_t* __restrict__ part_seg,
                                  int P, uint32_t* __restrict__ cstart,
                                  uint32_t* __restrict__ cend, uint32_t* __restrict__ cseg, uint64_t* __restrict__ ckey,
                                  uint32_t* __restrict__ cidx) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
        const uint64_t key = run_key[r];
        const uint32_t seg = (uint32_t)(key % S);
        // word-range part of the segment (exchange pipelining, W = 1): part_seg[j] = first segment of part j
        int part = 0;
        for (int j = 1; j < P; ++j) part += (seg >= part_seg[j]) ? 1 : 0;
        const uint64_t wave = (key / S) * (uint64_t)P + (uint64_t)part;
        const uint32_t off = run_off[r], len = run_len[r];
        uint32_t c = chunk_off[r];
        for (uint32_t s = 0; s < len; s += chunk, ++c) {
            const uint32_t e = min(s + chunk, len);
            cstart[c] = off + s;
            cend[c] = off + e;
            cseg[c] = seg;
            ckey[c] = wave * (uint64_t)(chunk + 1) + (uint64_t)(chunk - (e - s));
            cidx[c] = c;
        }
    }
}

__global__ void gather3_kernel(const uint32_t* __restrict__ idx, uint32_t n, const uint32_t* __restrict__ a,
                               const uint32_t* __restrict__ b, const uint32_t* __restrict__ c, uint32_t* __restrict__ ao,
                               uint32_t* __restrict__ bo, uint32_t* __restrict__ co) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t x = idx[j];
        ao[j] = a[x]; bo[j] = b[x]; co[j] = c[x];
    }
}

__global__ void seg_of_key_kernel(const uint64_t* __restrict__ key, uint32_t n, uint64_t S, uint32_t* __restrict__ seg) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        seg[j] = (uint32_t)(key[j] % S);
}

// doc index (local) of every sorted position, and 0..n-1 for the CSR sort
// doc -> sorted-positions CSR by counting: slot j of document d's range gets one of d's sorted positions.
// The order inside a document's range is arbitrary (atomics); its one consumer, the W = 1 recount, builds
// an order-independent histogram from it, so every count stays deterministic.
__global__ void csr_scatter_kernel(const uint32_t* __restrict__ tdoc, uint32_t n, const uint32_t* __restrict__ doc_ptr,
                                   uint32_t* __restrict__ cursor, uint32_t* __restrict__ doc_pos) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t d = tdoc[j];
        doc_pos[doc_ptr[d] + atomicAdd(cursor + d, 1u)] = j;
    }
}

__global__ void tdoc_kernel(const uint32_t* __restrict__ tok_id, uint32_t n, const int32_t* __restrict__ doc,
                            const int32_t* __restrict__ local_of_doc, uint32_t* __restrict__ tdoc,
                            uint32_t* __restrict__ q) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t d = doc[tok_id[j]];
        tdoc[j] = (uint32_t)(local_of_doc ? local_of_doc[d] : d);
        q[j] = j;
    }
}

}  // namespace spdp
