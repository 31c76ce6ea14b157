// Thin device-memory layer. The nvcc build (libfcsg.so) uses the CUDA
// runtime; the FCSG_EMULATE build used only by the CPU unit tests maps the
// same calls onto host memory.
#pragma once

#include <cstddef>
#include <string>

namespace fcsg {
namespace dev {

void set_device(int device);
// true exactly once per (flag, current device): per-device one-time setup such
// as cudaFuncSetAttribute (function attributes are per device). flag is a
// caller-owned word, one bit per device ordinal < 64; thread-safe.
bool first_on_device(unsigned long long* flag);
void* create_stream();
void destroy_stream(void* s);
// events for fork / join between streams (also inside graph capture)
void* create_event();
void destroy_event(void* e);
void record(void* event, void* stream);
void wait(void* stream, void* event);
void* alloc(size_t bytes);
void free(void* p);
void h2d(void* dst, const void* src, size_t bytes, void* stream);
void d2h(void* dst, const void* src, size_t bytes, void* stream);
// enqueue only (no stream sync)
void h2d_async(void* dst, const void* src, size_t bytes, void* stream);
void d2h_async(void* dst, const void* src, size_t bytes, void* stream);
void d2d(void* dst, const void* src, size_t bytes, void* stream);
void memset0(void* p, size_t bytes, void* stream);
void sync(void* stream);
void sync_device();
// throws Error(kCuda) if the last launch failed
void check(const char* what);
bool is_cuda();
// CUDA graph capture of everything enqueued on `stream` between begin and end
void graph_begin(void* stream);
void graph_end(void* stream, void** graph, void** exec);
void graph_launch(void* exec, void* stream);
void graph_destroy(void* exec, void* graph);
// elapsed milliseconds of work enqueued on `stream` by fn()
double time_on_stream(void* stream, void (*fn)(void*), void* arg);

template <class T>
T* alloc_n(size_t n) {
    return static_cast<T*>(alloc(n * sizeof(T)));
}

}  // namespace dev
}  // namespace fcsg
