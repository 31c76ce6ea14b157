#include "dev.h"

#include <cstdlib>
#include <cstring>

#include "fc_tables.h"
#include "fcsg_common.h"

namespace fcsg {
namespace dev {

#if FCSG_CUDA

namespace {
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

bool is_cuda() { return true; }
void set_device(int device) { ck(cudaSetDevice(device), "cudaSetDevice"); }
bool first_on_device(unsigned long long* flag) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    const unsigned long long old = __atomic_fetch_or(flag, bit, __ATOMIC_ACQ_REL);
    return (old & bit) == 0;
}
void* create_stream() {
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    return s;
}
void destroy_stream(void* s) { cudaStreamDestroy(static_cast<cudaStream_t>(s)); }
void* create_event() {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    return e;
}
void destroy_event(void* e) { cudaEventDestroy(static_cast<cudaEvent_t>(e)); }
void record(void* event, void* stream) {
    ck(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)), "event record");
}
void wait(void* stream, void* event) {
    ck(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0), "stream wait");
}
void* alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
    return p;
}
void free(void* p) {
    if (p) cudaFree(p);
}
void h2d(void* dst, const void* src, size_t bytes, void* stream) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)), "h2d");
    ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "h2d sync");
}
void d2h(void* dst, const void* src, size_t bytes, void* stream) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)), "d2h");
    ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "d2h sync");
}
void h2d_async(void* dst, const void* src, size_t bytes, void* stream) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)), "h2d");
}
void d2h_async(void* dst, const void* src, size_t bytes, void* stream) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)), "d2h");
}
void d2d(void* dst, const void* src, size_t bytes, void* stream) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)), "d2d");
}
void memset0(void* p, size_t bytes, void* stream) {
    ck(cudaMemsetAsync(p, 0, bytes, static_cast<cudaStream_t>(stream)), "memset");
}
void sync(void* stream) { ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "stream sync"); }
void sync_device() { ck(cudaDeviceSynchronize(), "device sync"); }
void check(const char* what) { ck(cudaGetLastError(), what); }
void graph_begin(void* stream) {
    ck(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream), cudaStreamCaptureModeThreadLocal), "capture");
}
void graph_end(void* stream, void** graph, void** exec) {
    cudaGraph_t g;
    ck(cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g), "end capture");
    cudaGraphExec_t x;
    ck(cudaGraphInstantiate(&x, g, 0), "graph instantiate");
    *graph = g;
    *exec = x;
}
void graph_launch(void* exec, void* stream) {
    ck(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), static_cast<cudaStream_t>(stream)), "graph launch");
}
void graph_destroy(void* exec, void* graph) {
    if (exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
    if (graph) cudaGraphDestroy(static_cast<cudaGraph_t>(graph));
}

double time_on_stream(void* stream, void (*fn)(void*), void* arg) {
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ck(cudaEventRecord(a, s), "record");
    fn(arg);
    ck(cudaEventRecord(b, s), "record");
    ck(cudaEventSynchronize(b), "event sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

#else

bool is_cuda() { return false; }
void set_device(int) {}
bool first_on_device(unsigned long long* flag) {
    const unsigned long long old = __atomic_fetch_or(flag, 1ull, __ATOMIC_ACQ_REL);
    return (old & 1ull) == 0;
}
void* create_stream() { return nullptr; }
void destroy_stream(void*) {}
void* create_event() { return nullptr; }
void destroy_event(void*) {}
void record(void*, void*) {}
void wait(void*, void*) {}
void* alloc(size_t bytes) { return std::calloc(bytes ? bytes : 16, 1); }
void free(void* p) { std::free(p); }
void h2d(void* dst, const void* src, size_t bytes, void*) { std::memcpy(dst, src, bytes); }
void d2h(void* dst, const void* src, size_t bytes, void*) { std::memcpy(dst, src, bytes); }
void d2d(void* dst, const void* src, size_t bytes, void*) { std::memmove(dst, src, bytes); }
void h2d_async(void* dst, const void* src, size_t bytes, void*) { std::memcpy(dst, src, bytes); }
void d2h_async(void* dst, const void* src, size_t bytes, void*) { std::memcpy(dst, src, bytes); }
void memset0(void* p, size_t bytes, void*) { std::memset(p, 0, bytes); }
void sync(void*) {}
void sync_device() {}
void check(const char*) {}
void graph_begin(void*) {}
void graph_end(void*, void**, void**) {}
void graph_launch(void*, void*) {}
void graph_destroy(void*, void*) {}
double time_on_stream(void*, void (*fn)(void*), void* arg) {
    fn(arg);
    return 0.0;
}

#endif

}  // namespace dev
}  // namespace fcsg
