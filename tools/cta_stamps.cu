// cta_stamps.cu -- diagnostics: per-CTA start / tables-filled and per-warp
// finish times (%globaltimer) of one C2 decrypt launch, to see where the
// per-launch overhead goes (launch ramp, table fill, tail).  Builds the
// kernels with -DKG_CTA_STAMPS by including their source.
#define KG_CTA_STAMPS 1
#include "../paper_1305_3345_b200/csrc/kg_kernels.cu"

#include <stdio.h>

int main(int argc, char **argv) {
    const bool enc = argc > 1 && argv[1][0] == 'e';  // "enc": C3 AES-256-CBC encrypt 1 GiB
    kg::BaseTables t;
    kg::build_base_tables(&t);
    if (kg::kernels_init(t) != cudaSuccess) return 1;
    uint8_t key[32] = {1, 2, 3, 4};
    kg::RoundKeys enc_k, dec_k;
    kg::expand_key(key, enc ? 32 : 16, &enc_k, &dec_k);
    const uint64_t n = enc ? 262144 : 65536, pb = 4096;
    uint8_t *in, *out, *iv;
    cudaMalloc(&in, n * pb);
    cudaMalloc(&out, n * pb);
    cudaMalloc(&iv, n * 16);
    cudaMemset(in, 7, n * pb);
    kg::LaunchArgs a;
    a.in = (const uint4 *)in;
    a.out = (uint4 *)out;
    a.ivs = (const uint4 *)iv;
    a.n_pages = n;
    a.m = pb / 16;
    a.in_place = 0;
    a.rk = enc ? enc_k : dec_k;
    for (int rep = 0; rep < 5; rep++) kg::launch_pages(enc ? 0 : 1, 0, enc ? 14 : 10, a, 148, 0);
    cudaDeviceSynchronize();
    static unsigned long long h[148 * 34];
    cudaMemcpyFromSymbol(h, kg::g_stamps, sizeof h);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 148; c++) t0 = h[c * 34] < t0 ? h[c * 34] : t0;
    printf("{\"cta\": [");
    for (int c = 0; c < 148; c++) {
        unsigned long long wmin = ~0ull, wmax = 0;
        for (int w = 0; w < 32; w++) {
            unsigned long long v = h[c * 34 + 2 + w];
            wmin = v < wmin ? v : wmin;
            wmax = v > wmax ? v : wmax;
        }
        printf("%s[%llu, %llu, %llu, %llu]", c ? ", " : "", h[c * 34] - t0, h[c * 34 + 1] - t0, wmin - t0, wmax - t0);
    }
    printf("]}\n");
    return 0;
}
