// Probe (tools only): can a green context's stream run runtime-API kernels on memory
// allocated in the primary context, with events recorded/waited across the two contexts?
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_add(int* p, int v) { p[threadIdx.x] += v; }
__global__ void __launch_bounds__(128) k_big(int* p) {
    extern __shared__ int sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    p[threadIdx.x] += sm[127 - threadIdx.x];
}

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("FAIL %s -> %d at %d\n", #x, (int)e_, __LINE__); } } while (0)

int main() {
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    int* d = nullptr;
    CK(cudaMalloc(&d, 128 * sizeof(int)));
    CK(cudaMemset(d, 0, 128 * sizeof(int)));
    CUcontext prim = nullptr;
    CK(cuCtxGetCurrent(&prim));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource full, part, rem;
    unsigned nb = 1;
    CK(cuDeviceGetDevResource(dev, &full, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs %u\n", full.sm.smCount);
    CK(cuDevSmResourceSplitByCount(&part, &nb, &full, &rem, 0, 128));
    printf("split: %u groups, part %u SMs, rem %u SMs\n", nb, part.sm.smCount, rem.sm.smCount);
    CUdevResourceDesc desc;
    CK(cuDevResourceGenerateDesc(&desc, &part, 1));
    CUgreenCtx g;
    CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUcontext gctx;
    CK(cuCtxFromGreenCtx(&gctx, g));
    CUstream gs;
    CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
    cudaStream_t ps;
    CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
    cudaEvent_t ev_prim;
    CK(cudaEventCreateWithFlags(&ev_prim, cudaEventDisableTiming));
    // 1. primary stream work, primary event, green stream waits on it (primary current)
    k_add<<<1, 128, 0, ps>>>(d, 1);
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev_prim, ps));
    CK(cudaStreamWaitEvent((cudaStream_t)gs, ev_prim, 0));
    // 2. launch on the green stream with the PRIMARY context current
    k_add<<<1, 128, 0, (cudaStream_t)gs>>>(d, 10);
    printf("launch green stream, primary current: %s\n", cudaGetErrorString(cudaGetLastError()));
    // 3. launch on the green stream with the GREEN context current
    CK(cuCtxSetCurrent(gctx));
    k_add<<<1, 128, 0, (cudaStream_t)gs>>>(d, 100);
    printf("launch green stream, green current: %s\n", cudaGetErrorString(cudaGetLastError()));
    // big smem kernel needs the attribute in this context
    printf("attr in green: %s\n", cudaGetErrorString(cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024)));
    k_big<<<1, 128, 100 * 1024, (cudaStream_t)gs>>>(d);
    printf("big smem launch green: %s\n", cudaGetErrorString(cudaGetLastError()));
    // primary event recorded on the green stream (green current)
    printf("record primary event on green stream: %s\n", cudaGetErrorString(cudaEventRecord(ev_prim, (cudaStream_t)gs)));
    cudaEvent_t ev_green;
    CK(cudaEventCreateWithFlags(&ev_green, cudaEventDisableTiming));
    printf("record green event on green stream: %s\n", cudaGetErrorString(cudaEventRecord(ev_green, (cudaStream_t)gs)));
    CK(cuCtxSetCurrent(prim));
    printf("primary stream waits green event: %s\n", cudaGetErrorString(cudaStreamWaitEvent(ps, ev_green, 0)));
    printf("primary stream waits primary event (recorded on green): %s\n", cudaGetErrorString(cudaStreamWaitEvent(ps, ev_prim, 0)));
    k_add<<<1, 128, 0, ps>>>(d, 1000);
    CK(cudaGetLastError());
    printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    CK(cuCtxSetCurrent(gctx));
    printf("green ctx sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    CK(cuCtxSetCurrent(prim));
    int h[128];
    CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    printf("h[0]=%d h[5]=%d (expect 1+10?+100+127+1000 / +122)\n", h[0], h[5]);
    return 0;
}
