// Mechanism probe: two processes on the same GPU exchange data through CUDA-IPC-mapped buffers with
// epoch flags (system-scope release / acquire), inside a CUDA graph, for E epochs.
//   p2p_probe <rank> <dir>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unistd.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("rank %d: %s failed: %s\n", rank, #x, cudaGetErrorString(e_)); return 1; } } while (0)
static int rank;
struct Win { double data[2][4096]; unsigned long long flag[2]; };
__global__ void k_put(Win* peer, const unsigned long long* epoch, int me) {
    const unsigned long long e = *epoch;
    const int par = (int)(e & 1);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) peer->data[par][i] = me * 1e6 + (double)e * 10 + i * 1e-3;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(&peer->flag[me]), "l"(e) : "memory");
    }
}
__global__ void k_wait_check(Win* mine, unsigned long long* epoch, int other, int* bad) {
    const unsigned long long e = *epoch;
    __shared__ int ok;
    if (threadIdx.x == 0) {
        unsigned long long f = 0; long spins = 0;
        do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(&mine->flag[other]) : "memory"); ++spins; }
        while (f < e && spins < (1L << 34));
        ok = f >= e;
    }
    __syncthreads();
    const int par = (int)(e & 1);
    int nb = ok ? 0 : 100000;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        if (mine->data[par][i] != other * 1e6 + (double)e * 10 + i * 1e-3) ++nb;
    if (nb) atomicAdd(bad, nb);
    __syncthreads();
    if (threadIdx.x == 0) *epoch = e + 1;
}
int main(int argc, char** argv) {
    rank = atoi(argv[1]);
    std::string dir = argv[2];
    const int other = 1 - rank, E = argc > 3 ? atoi(argv[3]) : 200;
    CK(cudaSetDevice(0));
    Win* w; CK(cudaMalloc(&w, sizeof(Win))); CK(cudaMemset(w, 0, sizeof(Win)));
    unsigned long long* ep; CK(cudaMalloc(&ep, 8));
    unsigned long long one = 1; CK(cudaMemcpy(ep, &one, 8, cudaMemcpyHostToDevice));
    int* bad; CK(cudaMalloc(&bad, 4)); CK(cudaMemset(bad, 0, 4));
    cudaIpcMemHandle_t h; CK(cudaIpcGetMemHandle(&h, w));
    { std::string f = dir + "/h" + std::to_string(rank); FILE* fp = fopen((f + ".tmp").c_str(), "wb"); fwrite(&h, sizeof(h), 1, fp); fclose(fp); rename((f + ".tmp").c_str(), f.c_str()); }
    cudaIpcMemHandle_t ph; std::string pf = dir + "/h" + std::to_string(other);
    for (;;) { FILE* fp = fopen(pf.c_str(), "rb"); if (fp) { size_t n = fread(&ph, sizeof(ph), 1, fp); fclose(fp); if (n == 1) break; } usleep(10000); }
    Win* peer; CK(cudaIpcOpenMemHandle((void**)&peer, ph, cudaIpcMemLazyEnablePeerAccess));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    k_put<<<1, 256, 0, s>>>(peer, ep, rank);
    k_wait_check<<<1, 256, 0, s>>>(w, ep, other, bad);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int e = 0; e < E; ++e) CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(b, s);
    CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, a, b);
    int hb = -1; CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    printf("rank %d: %d epochs, bad=%d, %.3f ms per epoch\n", rank, E, hb, ms / E);
    CK(cudaIpcCloseMemHandle(peer));
    return hb != 0;
}
