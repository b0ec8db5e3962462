// pgl_pack.cu — step records built on the device from compact GFA steps.
//
// pgl_graph_create_gfa parses a GFA into node lengths and one u32 word per
// path step (node | reverse << 31: 4 bytes instead of the reference's 24-byte
// PathStep) and uploads those; the device then does build_graph's offset
// pass (graph.cpp:38-50) and path_position (graph.hpp:98-109): gather each
// step's node length, exclusive-scan them (CUB) in chunks of 2^30 with a
// carried total, subtract the scan value at the path's first step, and
// write the 16-byte step records with both endpoint positions.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr uint64_t kScanChunk = 1ULL << 30;

__global__ void k_gather_len(const uint32_t* __restrict__ steps, const uint32_t* __restrict__ node_len,
                             uint64_t* __restrict__ out, uint64_t b, uint64_t e) {
    for (uint64_t k = b + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < e;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[k] = __ldg(node_len + (__ldg(steps + k) & 0x7FFFFFFFu));
}

__global__ void k_add_carry(uint64_t* __restrict__ offs, uint64_t b, uint64_t e, const uint64_t* __restrict__ carry) {
    const uint64_t c = *carry;
    for (uint64_t k = b + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < e;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        offs[k] += c;
}

__global__ void k_next_carry(const uint64_t* __restrict__ offs, const uint32_t* __restrict__ steps,
                             const uint32_t* __restrict__ node_len, uint64_t last, uint64_t* __restrict__ carry) {
    *carry = offs[last] + node_len[steps[last] & 0x7FFFFFFFu];
}

__global__ void k_build_records(const uint32_t* __restrict__ steps, const uint32_t* __restrict__ node_len,
                                const uint64_t* __restrict__ offs, const uint64_t* __restrict__ cum, uint32_t P,
                                uint64_t S, StepRec* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < S;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t lo = 0, hi = P;  // path of step k
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(cum + mid) <= k)
                lo = mid;
            else
                hi = mid;
        }
        const uint32_t w = __ldg(steps + k);
        const uint32_t node = w & 0x7FFFFFFFu;
        const uint64_t off = offs[k] - offs[__ldg(cum + lo)];  // PathStep.offset
        const uint64_t len = __ldg(node_len + node);
        const uint64_t ps = (w >> 31) ? off + len : off;      // path_position(start)
        const uint64_t pe = (w >> 31) ? off : off + len;      // path_position(end)
        out[k] = StepRec{node, static_cast<uint32_t>(ps), static_cast<uint32_t>(pe),
                         static_cast<uint32_t>((ps >> 32) | ((pe >> 32) << 16))};
    }
}

// 8-byte records (DevGraph::rec8): step gi of path p goes to gi + p; the
// path's sentinel after its last step carries the far end position. For a
// forward step pos_start = offset < pos_end, for a reverse one the other
// way round (path_position, graph.hpp:98-109), so the orientation is
// pos_start > pos_end and the step's offset is the smaller of the two.
__global__ void k_build_rec8(const StepRec* __restrict__ step, const uint64_t* __restrict__ cum, uint32_t P,
                             uint64_t S, uint2* __restrict__ out) {
    for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; gi < S;
         gi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t lo = 0, hi = P;  // largest p with cum[p] <= gi
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cum[mid] <= gi) lo = mid; else hi = mid;
        }
        const StepRec r = step[gi];
        const bool rev = r.ps_lo > r.pe_lo;
        out[gi + lo] = make_uint2(r.node | (rev ? 0x80000000u : 0u), rev ? r.pe_lo : r.ps_lo);
        if (gi + 1 == cum[lo + 1]) out[gi + lo + 1] = make_uint2(0u, rev ? r.ps_lo : r.pe_lo);
    }
}

}  // namespace

void build_rec8_device(const StepRec* step, const uint64_t* cum, uint32_t P, uint64_t S, uint2* out,
                       cudaStream_t stream) {
    k_build_rec8<<<148 * 16, 256, 0, stream>>>(step, cum, P, S, out);
    PGL_CUDA(cudaGetLastError());
}

void build_records_device(const uint32_t* d_steps, const uint32_t* d_node_len, const uint64_t* d_cum, uint32_t P,
                          uint64_t S, StepRec* d_out, void* stream_) {
    cudaStream_t s = static_cast<cudaStream_t>(stream_);
    if (S == 0) return;
    uint64_t* offs = nullptr;
    uint64_t* carry = nullptr;
    PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&offs), S * sizeof(uint64_t), s));
    PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&carry), sizeof(uint64_t), s));
    PGL_CUDA(cudaMemsetAsync(carry, 0, sizeof(uint64_t), s));
    size_t temp_bytes = 0;
    PGL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, offs, offs,
                                           static_cast<int>(std::min<uint64_t>(S, kScanChunk)), s));
    void* temp = nullptr;
    PGL_CUDA(cudaMallocAsync(&temp, std::max<size_t>(temp_bytes, 1), s));
    int dev = 0, sms = 0;
    PGL_CUDA(cudaGetDevice(&dev));
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = static_cast<unsigned>(sms * 8);
    for (uint64_t b = 0; b < S; b += kScanChunk) {
        const uint64_t e = std::min<uint64_t>(S, b + kScanChunk);
        k_gather_len<<<grid, 256, 0, s>>>(d_steps, d_node_len, offs, b, e);
        PGL_CUDA(cudaGetLastError());
        PGL_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, offs + b, offs + b, static_cast<int>(e - b), s));
        k_add_carry<<<grid, 256, 0, s>>>(offs, b, e, carry);
        k_next_carry<<<1, 1, 0, s>>>(offs, d_steps, d_node_len, e - 1, carry);
        PGL_CUDA(cudaGetLastError());
    }
    k_build_records<<<grid, 256, 0, s>>>(d_steps, d_node_len, offs, d_cum, P, S, d_out);
    PGL_CUDA(cudaGetLastError());
    PGL_CUDA(cudaFreeAsync(temp, s));
    PGL_CUDA(cudaFreeAsync(offs, s));
    PGL_CUDA(cudaFreeAsync(carry, s));
}

}  // namespace pgl
