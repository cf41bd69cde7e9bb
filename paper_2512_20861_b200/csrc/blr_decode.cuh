// blr_decode.cuh -- constants of the small-token (decode, n_tok <= DECODE_MAX_TOKENS) path (SURVEY
// §8 row f2; §3.1: at small n the layer is bound by reading its factors, not by
// FLOPs) and its one non-GEMM kernel.  The weight-streaming stages themselves are the tensor-core
// decode_tc_kernel of blr_decode_tc.cuh.
//
//   decode_s2_kernel : BLAST S2, Z''[k][t][rho] = sum_l S[l,k,rho] Z[l][t][rho]  (fp32), used when
//                      the S1 + S2 cluster kernel does not apply (p > 1024 or b1 with no cluster
//                      factorisation <= 8 x 4).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx.cuh"

namespace blr {

constexpr int DECODE_MAX_TOKENS = 16;
constexpr int DECODE_THREADS = 256;

// BLAST S2 for the decode path: Z''[k][t][rho] = sum_l S[l,k,rho] * Z[l][t][rho], fp32 in/out.
__global__ void __launch_bounds__(DECODE_THREADS)
    decode_s2_kernel(const float* __restrict__ Z, const __nv_bfloat16* __restrict__ S, float* __restrict__ Zpp,
                     int n_tok, int b1, int b2, int r) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long total = static_cast<long long>(b2) * n_tok * r;
    for (long long e = blockIdx.x * static_cast<long long>(DECODE_THREADS) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * DECODE_THREADS) {
        const int rho = static_cast<int>(e % r);
        const long long kt = e / r;
        const int t = static_cast<int>(kt % n_tok);
        const int k = static_cast<int>(kt / n_tok);
        float s = 0.f;
        for (int l = 0; l < b1; ++l)
            s = fmaf(__bfloat162float(S[(static_cast<long long>(l) * b2 + k) * r + rho]),
                     Z[(static_cast<long long>(l) * n_tok + t) * r + rho], s);
        Zpp[e] = s;
    }
}

}  // namespace blr
