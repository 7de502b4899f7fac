// bv_probe.cu — phase timing of the bitvector kernel in isolation at N=1 (design input).
#include "../paper_1909_11150_b200/csrc/gr_kernels.cu"
#include <cstdio>
#include <vector>
using namespace gr;
int main(int argc, char **argv) {
    const int T = 68, G = 10, W = (T + 2 + 31) / 32, nbits = T + 2;
    std::vector<int> gob(W * 32, -1), tob(W * 32, -1), gbb(G), gbe(G), gn(G, 1);
    std::vector<int64_t> ge(G, 100);
    for (int b = 2; b < nbits; ++b) { tob[b] = b - 2; gob[b] = (b - 2) * G / T; }
    for (int g = 0; g < G; ++g) { gbb[g] = 1 << 30; gbe[g] = -1; }
    for (int b = 2; b < nbits; ++b) { gbb[gob[b]] = std::min(gbb[gob[b]], b); gbe[gob[b]] = std::max(gbe[gob[b]], b + 1); }
    auto up = [](auto &v) { void *d; cudaMalloc(&d, v.size() * sizeof(v[0])); cudaMemcpy(d, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice); return d; };
    BvParams p{};
    p.group_of_bit = (int *)up(gob); p.tensor_of_bit = (int *)up(tob); p.group_bit_begin = (int *)up(gbb);
    p.group_bit_end = (int *)up(gbe); p.group_nchunks = (int *)up(gn); p.group_elems = (int64_t *)up(ge);
    cudaMalloc(&p.group_rel_epoch, 4 * G); cudaMemset(p.group_rel_epoch, 0, 4 * G);
    uint32_t *flags; cudaMalloc(&flags, 4 * W * 32); cudaMemset(flags, 0, 4 * W * 32); p.dev_flags = flags;
    uint64_t *slot; cudaMalloc(&slot, 16 * W); p.slot[0] = slot;
    cudaMalloc(&p.out_released, 4 * G); cudaMalloc(&p.out_cum, 4 * (G + 1));
    HostResult *h; size_t rb = sizeof(HostResult) + 4 * W + 4 * G;
    cudaHostAlloc(&h, rb, cudaHostAllocMapped); HostResult *d; cudaHostGetDevicePointer((void **)&d, h, 0);
    p.result = d; p.T = T; p.G = G; p.W = W; p.nbits = nbits; p.rank = 0; p.N = 1; p.timeout_ns = 1000000000ull;
    p.use_inline = 1;
    // big buffer to thrash L2 between launches
    char *junk; size_t jb = 512ull << 20; cudaMalloc(&junk, jb);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int thrash = 0; thrash < 2; ++thrash) {
        double a = 0, b = 0, c = 0, tot = 0; int n = 200;
        for (int i = 0; i < n + 20; ++i) {
            p.epoch = i + 1; p.tag = i + 1; p.parity = i & 1; p.seq = 1000 * thrash + i + 1;
            for (int w = 0; w < W; ++w) p.inline_bits[w] = 0xffffffffu;
            if (thrash) cudaMemsetAsync(junk, i, jb, s);
            launch_bitvector(p, s);
            while (h->seq != p.seq) {}
            if (i >= 20) { a += (h->t_populated - h->t_start) / 1e3; b += (h->t_anded - h->t_populated) / 1e3; c += (h->t_end - h->t_anded) / 1e3; tot += (h->t_end - h->t_start) / 1e3; }
            cudaStreamSynchronize(s);
        }
        printf("threads=%d batch=%d thrashL2=%d: populate %.2f  AND %.2f  release %.2f  total %.2f us\n", BV_THREADS, BV_BATCH, thrash, a / n, b / n, c / n, tot / n);
    }
    return 0;
}
