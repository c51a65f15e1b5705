// Probe: does programmatic dependent launch (PDL) let kernel B's CTAs fill the
// SMs kernel A's tail leaves idle, and does an event record / stream wait placed
// between A and B keep or break that overlap?  One CTA per SM (big smem), A's
// CTAs spin for uneven times, B starts with no griddepcontrol.wait (its work is
// independent of A) and waits at its end (so B's completion implies A's).
// Prints, per case, B's first CTA start minus A's last CTA end (negative =
// overlap) and the A-start -> B-end span.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/pdl_probe tools/pdl_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin_kernel(unsigned long long* start, unsigned long long* end, int base_us,
                            int pdl_role) {
  extern __shared__ char smem[];
  if (pdl_role & 1) asm volatile("griddepcontrol.launch_dependents;");
  const unsigned long long t0 = gtime();
  const unsigned long long dur = (unsigned long long)(base_us + (blockIdx.x * 37) % 23 * 10) * 1000ull;
  if (threadIdx.x == 0) smem[0] = 1;
  while (gtime() - t0 < dur) {
  }
  if (pdl_role & 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    start[blockIdx.x] = t0;
    end[blockIdx.x] = gtime() + smem[0] - 1;
  }
}

__global__ void stamp_kernel(unsigned long long* t) {
  if (threadIdx.x == 0) t[0] = gtime();
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem = 200 * 1024;
  CK(cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int n = sms * 3 + sms / 3;  // a ragged last wave
  unsigned long long *as, *ae, *bs, *be;
  CK(cudaMalloc(&as, n * 8));
  CK(cudaMalloc(&ae, n * 8));
  CK(cudaMalloc(&bs, n * 8));
  CK(cudaMalloc(&be, n * 8));
  unsigned long long* cs;
  CK(cudaMalloc(&cs, 8));
  cudaStream_t s, s2;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t ev, done;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(done, s2));
  CK(cudaStreamSynchronize(s2));
  const char* names[] = {"no PDL", "PDL adjacent", "PDL + event record between",
                         "PDL + wait(completed event) between", "PDL + wait(other stream event) between"};
  for (int rep = 0; rep < 2; ++rep)
    for (int c = 0; c < 5; ++c) {
      spin_kernel<<<n, 128, smem, s>>>(as, ae, 100, c ? 1 : 0);
      if (c == 2) CK(cudaEventRecord(ev, s));
      if (c == 3) CK(cudaStreamWaitEvent(s, done, 0));
      if (c == 4) {
        CK(cudaEventRecord(ev, s2));
        CK(cudaStreamWaitEvent(s, ev, 0));
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = c ? 1 : 0;
      CK(cudaLaunchKernelEx(&cfg, spin_kernel, bs, be, 100, c ? 2 : 0));
      if (c == 2) {  // when does the event between A and B fire: at A's completion?
        CK(cudaStreamWaitEvent(s2, ev, 0));
        stamp_kernel<<<1, 32, 0, s2>>>(cs);
      }
      CK(cudaStreamSynchronize(s));
      CK(cudaStreamSynchronize(s2));
      std::vector<unsigned long long> a0(n), a1(n), b0(n), b1(n);
      CK(cudaMemcpy(a0.data(), as, n * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(a1.data(), ae, n * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b0.data(), bs, n * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b1.data(), be, n * 8, cudaMemcpyDeviceToHost));
      unsigned long long amin = ~0ull, amax = 0, bmin = ~0ull, bmax = 0;
      for (int i = 0; i < n; ++i) {
        amin = a0[i] < amin ? a0[i] : amin;
        amax = a1[i] > amax ? a1[i] : amax;
        bmin = b0[i] < bmin ? b0[i] : bmin;
        bmax = b1[i] > bmax ? b1[i] : bmax;
      }
      unsigned long long cst = 0;
      CK(cudaMemcpy(&cst, cs, 8, cudaMemcpyDeviceToHost));
      if (rep && c == 2)
        printf("  event waiter start - A.last_end = %8.1f us (must be >= 0)\n",
               ((double)cst - (double)amax) / 1e3);
      if (rep)
        printf("%-40s B.first_start - A.last_end = %8.1f us   span = %8.1f us\n", names[c],
               ((double)bmin - (double)amax) / 1e3, (double)(bmax - amin) / 1e3);
    }
  return 0;
}
