// gather_ceiling.cu -- measurement tool (not the product): the ceiling of the SpMM's access pattern on this GPU.
//
// The aggregation (a6 / a10) is a stream of row gathers: for every kept edge, one row of
// d * s bytes (16-byte vectors, one per lane) from a source buffer that is L2-resident when the working set fits the
// 126 MB L2 (the Reddit-shaped hidden layers at m = 1: 119 MB; every layer at m = 8) and DRAM-resident otherwise.
// This kernel does exactly that access pattern with nothing else: warps walk a random column list, each lane keeps
// U = 8 independent 16-byte non-coherent loads in flight (the SpMM's register double issue), and XOR-folds them so
// the loads cannot be removed.  Its GB/s over (rows, width, working set, index distribution) is the roofline the
// SpMM's algorithmic bytes are divided by in bench.py ("ceiling"), next to the HBM copy peak.
//
//   gather_ceiling [iters]                                   synthetic cases (uniform / skewed column streams)
//   gather_ceiling iters colfile row_bytes stride_bytes name  the column stream of a real induced CSR (int32 file),
//                                                             e.g. the Reddit-shaped R-MAT graph in CSR order
// -> one JSON line per case on stdout
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int U = 8;

// each warp owns edges [w*chunk, (w+1)*chunk); a row of nvec 16-byte vectors (nvec <= 32) is read by nvec lanes, so
// 32 / nvec lane groups take alternate edges (the SpMM's narrow-row layout)
__global__ void __launch_bounds__(256) k_gather(const uint4* __restrict__ src, int nvec, int64_t ldv,
                                                const int32_t* __restrict__ col, int64_t nnz, int64_t chunk,
                                                uint4* __restrict__ sink) {
    const int lane = threadIdx.x & 31;
    const int G = 32 / nvec, grp = lane / nvec, vec = lane % nvec;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t e0 = w * chunk, e1 = min(nnz, e0 + chunk);
    uint4 acc = make_uint4(0, 0, 0, 0);
    int64_t e = grp < G ? e0 + grp : e1;   // nvec not dividing 32: the last 32 % nvec lanes idle
    for (; e + (int64_t)(U - 1) * G < e1; e += (int64_t)U * G) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int32_t c = __ldg(col + e + (int64_t)k * G);
            const uint4* p = src + (int64_t)c * ldv + vec;
            asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                         : "l"(p));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            acc.x ^= v[k].x; acc.y ^= v[k].y; acc.z ^= v[k].z; acc.w ^= v[k].w;
        }
    }
    for (; e < e1; e += G) {
        const uint4 v = __ldg(src + (int64_t)col[e] * ldv + vec);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x | acc.y | acc.z | acc.w) == 0x9E3779B9u) sink[threadIdx.x] = acc;   // practically never taken
}

// sequential read of the whole buffer (L2-resident re-read when it fits): the streaming reference
__global__ void k_stream(const uint4* __restrict__ src, int64_t n, uint4* __restrict__ sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(src + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x | acc.y | acc.z | acc.w) == 0x9E3779B9u) sink[threadIdx.x] = acc;
}

static double time_gather(const uint4* src, int nvec, int64_t ldv, const int32_t* d_col, int64_t nnz, int sms,
                          int iters, uint4* sink) {
    // one resident wave of 8 blocks x 8 warps per SM, equal edge chunks
    const int64_t warps = (int64_t)sms * 8 * 8;
    const int64_t chunk = (nnz + warps - 1) / warps;
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_gather<<<grid, 256>>>(src, nvec, ldv, d_col, nnz, chunk, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < iters; ++i) k_gather<<<grid, 256>>>(src, nvec, ldv, d_col, nnz, chunk, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
    return ms / 1e3 / iters;
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 20;
    int sms = 0, l2 = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    const int64_t nnz = 64ll << 20;   // 64 M gathered rows per launch
    struct Case { const char* name; int64_t rows; int width_b; int dist; };
    // dist 0: uniform random rows; 1: skewed (R-MAT-like: half the edges hit the first 1 % of rows)
    std::vector<Case> cases = {
        {"L2 16MB 512B uniform", 32768, 512, 0},   {"L2 64MB 512B uniform", 131072, 512, 0},
        {"L2 119MB 512B uniform", 232965, 512, 0}, {"L2 119MB 512B skewed", 232965, 512, 1},
        {"L2 23MB 512B uniform (m=8 hidden)", 44732, 512, 0},
        {"L2 64MB 128B uniform", 524288, 128, 0},  {"DRAM 1GB 512B uniform", 2097152, 512, 0},
        {"DRAM 1GB 512B skewed", 2097152, 512, 1}, {"DRAM 2.5GB 256B uniform (products L1)", 9796116, 256, 0},
    };
    uint4* sink;
    CK(cudaMalloc(&sink, 4096 * sizeof(uint4)));
    if (argc > 5) {   // file mode: a real column stream
        FILE* f = fopen(argv[2], "rb");
        if (!f) { fprintf(stderr, "cannot open %s\n", argv[2]); return 1; }
        fseek(f, 0, SEEK_END);
        const int64_t n = ftell(f) / 4;
        fseek(f, 0, SEEK_SET);
        std::vector<int32_t> c(n);
        if ((int64_t)fread(c.data(), 4, n, f) != n) { fprintf(stderr, "short read\n"); return 1; }
        fclose(f);
        int32_t mx = 0;
        for (int32_t x : c) mx = std::max(mx, x);
        const int row_bytes = atoi(argv[3]), stride = atoi(argv[4]);
        const int64_t rows = (int64_t)mx + 1, bytes = rows * stride;
        uint4* src;
        CK(cudaMalloc(&src, bytes));
        CK(cudaMemset(src, 1, bytes));
        int32_t* dc;
        CK(cudaMalloc(&dc, n * 4));
        CK(cudaMemcpy(dc, c.data(), n * 4, cudaMemcpyHostToDevice));
        const double t = time_gather(src, row_bytes / 16, stride / 16, dc, n, sms, iters, sink);
        printf("{\"case\": \"%s\", \"rows\": %lld, \"row_bytes\": %d, \"row_stride_bytes\": %d, "
               "\"working_set_bytes\": %lld, \"l2_bytes\": %d, \"gathered_rows\": %lld, \"gather_gbs\": %.1f, "
               "\"gather_plus_index_gbs\": %.1f, \"ms_per_launch\": %.4f}\n",
               argv[5], (long long)rows, row_bytes, stride, (long long)(rows * row_bytes), l2, (long long)n,
               (double)n * row_bytes / t / 1e9, (double)n * (row_bytes + 4) / t / 1e9, t * 1e3);
        return 0;
    }
    int32_t* d_col;
    CK(cudaMalloc(&d_col, nnz * sizeof(int32_t)));
    std::mt19937_64 rng(12345);
    std::vector<int32_t> col(nnz);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (const Case& cs : cases) {
        const int nvec = cs.width_b / 16;
        const int64_t bytes = cs.rows * cs.width_b;
        uint4* src;
        CK(cudaMalloc(&src, bytes));
        CK(cudaMemset(src, 1, bytes));
        const int64_t hot = std::max<int64_t>(1, cs.rows / 100);
        for (int64_t e = 0; e < nnz; ++e) {
            uint64_t r = rng();
            if (cs.dist == 1 && (r & 1)) col[e] = (int32_t)((r >> 1) % hot);
            else col[e] = (int32_t)((r >> 1) % cs.rows);
        }
        CK(cudaMemcpy(d_col, col.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
        const double t = time_gather(src, nvec, nvec, d_col, nnz, sms, iters, sink);
        const double gathered = (double)nnz * cs.width_b, idx = (double)nnz * 4;
        k_stream<<<sms * 8, 256>>>(src, bytes / 16, sink);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int i = 0; i < iters; ++i) k_stream<<<sms * 8, 256>>>(src, bytes / 16, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms2 = 0.f;
        CK(cudaEventElapsedTime(&ms2, a, b));
        const double t2 = ms2 / 1e3 / iters;
        printf("{\"case\": \"%s\", \"rows\": %lld, \"row_bytes\": %d, \"working_set_bytes\": %lld, \"l2_bytes\": %d, "
               "\"gathered_rows\": %lld, \"gather_gbs\": %.1f, \"gather_plus_index_gbs\": %.1f, "
               "\"stream_read_gbs\": %.1f, \"ms_per_launch\": %.4f}\n",
               cs.name, (long long)cs.rows, cs.width_b, (long long)bytes, l2, (long long)nnz, gathered / t / 1e9,
               (gathered + idx) / t / 1e9, (double)bytes / t2 / 1e9, t * 1e3);
        fflush(stdout);
        CK(cudaFree(src));
    }
    return 0;
}
