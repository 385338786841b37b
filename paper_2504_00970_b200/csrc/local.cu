// local.cu -- SURVEY 8(f) NEXT-2: the decode-side local segment and context growth (reading A29).
//
// P:456 (Sec. 4.2): "After generating the next token, we append its query to Q_s and repeat the
// process.  When a new sentence boundary ... is detected, we reset Q_s".  The generated tokens' K/V
// live in a ctx-owned HBM store per (sequence, layer, KV head).  The tokens of the sentence being
// generated form the local segment: always attended, not charged to tau.  When
// that sentence ends (its last token is a boundary -- the same event that resets Q_s, A11) it grows
// the context: at the next append it becomes a retrievable bucket like a prompt sentence (Eq. 1 mean
// of its keys appended to the layer's embeddings, its rows L + [start, end) appended to the layer's
// bucket offsets).  Everything is updated on the device, so a captured decode step replays.
//
// Per (layer, b) state gstat[b] = {generated count, start of the current sentence, sentence ended
// at the last token, overflow}.
#include "device_util.cuh"
#include "skv_internal.cuh"

namespace skv {
namespace {

// Grid (G, B).  Close the sentence that ended at the previous token (Eq. 1 over its keys, canonical
// order as compress_kernel / skvref_embed: fp32 sum in token order, one IEEE division, bf16 RNE),
// then store this step's k, v at the end of the store.  Reads gstat only; gen_state_kernel (next on
// the stream) advances it.
template <int D>
__global__ void __launch_bounds__(128) gen_close_append_kernel(const __nv_bfloat16* __restrict__ k,
                                                              const __nv_bfloat16* __restrict__ v,
                                                              __nv_bfloat16* __restrict__ Kg,
                                                              __nv_bfloat16* __restrict__ Vg, int max_gen,
                                                              const int32_t* __restrict__ gstat,
                                                              const int32_t* __restrict__ gS, int Smax,
                                                              __nv_bfloat16* __restrict__ E) {
    const int g = blockIdx.x, b = blockIdx.y, G = gridDim.x;
    const int n = gstat[b * 4 + 0], hot = gstat[b * 4 + 1], pend = gstat[b * 4 + 2];
    const size_t u = (size_t)b * G + g;
    const __nv_bfloat16* Ku = Kg + u * max_gen * D;
    if (pend && threadIdx.x < D / 8) {  // new bucket: mean of the sentence's keys
        const int l = threadIdx.x;
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        for (int t = hot; t < n; ++t) {
            float f[8];
            unpack8(reinterpret_cast<const uint4*>(Ku + (size_t)t * D)[l], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
        }
        const float c = (float)(n - hot);
        uint4 o;
        o.x = pack_bf16x2_rn(__fdiv_rn(acc[0], c), __fdiv_rn(acc[1], c));
        o.y = pack_bf16x2_rn(__fdiv_rn(acc[2], c), __fdiv_rn(acc[3], c));
        o.z = pack_bf16x2_rn(__fdiv_rn(acc[4], c), __fdiv_rn(acc[5], c));
        o.w = pack_bf16x2_rn(__fdiv_rn(acc[6], c), __fdiv_rn(acc[7], c));
        reinterpret_cast<uint4*>(E + (u * Smax + gS[b]) * D)[l] = o;
    }
    if (n < max_gen && threadIdx.x < D / 8) {
        const int l = threadIdx.x;
        reinterpret_cast<uint4*>(Kg + (u * max_gen + n) * D)[l] = reinterpret_cast<const uint4*>(k + u * D)[l];
        reinterpret_cast<uint4*>(Vg + (u * max_gen + n) * D)[l] = reinterpret_cast<const uint4*>(v + u * D)[l];
    }
}

// One thread per sequence: bucket offsets / count of a closed sentence, then the counters.
__global__ void gen_state_kernel(int B, int L, int max_gen, int tau, int32_t* __restrict__ gstat, int32_t* __restrict__ goff,
                                 int off_stride, int32_t* __restrict__ gS, const int32_t* __restrict__ input_token,
                                 const int32_t* __restrict__ bset, int nb, int32_t* __restrict__ gsid, int sid_stride,
                                 const int32_t* __restrict__ S_prompt, const int32_t* __restrict__ gS0) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int32_t* st = gstat + b * 4;
    const int n = st[0];
    if (st[2]) {  // the sentence [hot, n) is a bucket now: rows L + hot .. L + n
        const int s = gS[b];
        goff[(size_t)b * off_stride + s + 1] = L + n;
        gS[b] = s + 1;
        // retention: bucket ids map to sentence ids; a generated sentence is sentence S + k of the text
        if (gsid) gsid[(size_t)b * sid_stride + s] = S_prompt[b] + (s - gS0[b]);
        st[1] = n;
        st[2] = 0;
    }
    if (n < max_gen) {
        st[0] = n + 1;
        // this token ends the sentence (a boundary, A11), or the sentence reached tau tokens (the A5
        // cap, which also bounds the local segment by tau)
        st[2] = (in_set(input_token[b], bset, nb) || n + 1 - st[1] >= tau) ? 1 : 0;
    } else {
        st[3] = 1;  // overflow: the token was not stored (surfaced by sentencekv_sync)
    }
}

// SURVEY 8(e) fused gather: one thread advances the expected arrival count of this step and spins
// (acquire, system scope) until every rank's units have counted their arrival in this rank's buffer.
__global__ void wait_peers_kernel(const unsigned int* __restrict__ flag, unsigned int* __restrict__ target,
                                  unsigned int per_step) {
    if (threadIdx.x != 0) return;
    const unsigned int want = *target + per_step;
    *target = want;
    unsigned int v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if ((int)(v - want) >= 0) break;
        __nanosleep(64);
    }
}

}  // namespace

cudaError_t launch_wait_peers(const unsigned int* flag, unsigned int* target, unsigned int per_step, cudaStream_t st) {
    wait_peers_kernel<<<1, 32, 0, st>>>(flag, target, per_step);
    return cudaGetLastError();
}

cudaError_t launch_gen_append(const __nv_bfloat16* k, const __nv_bfloat16* v, __nv_bfloat16* Kg, __nv_bfloat16* Vg,
                              int max_gen, int32_t* gstat, int32_t* goff, int off_stride, int32_t* gS, int Smax,
                              __nv_bfloat16* E, const int32_t* input_token, const int32_t* bset, int nb, int B, int G,
                              int L, int d, int tau, int32_t* gsid, const int32_t* S_prompt, const int32_t* gS0,
                              cudaStream_t st) {
    if (d == 128)
        gen_close_append_kernel<128><<<dim3(G, B), 128, 0, st>>>(k, v, Kg, Vg, max_gen, gstat, gS, Smax, E);
    else
        gen_close_append_kernel<64><<<dim3(G, B), 128, 0, st>>>(k, v, Kg, Vg, max_gen, gstat, gS, Smax, E);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    gen_state_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, L, max_gen, tau, gstat, goff, off_stride, gS, input_token, bset,
                                                     nb, gsid, Smax, S_prompt, gS0);
    return cudaGetLastError();
}

}  // namespace skv
