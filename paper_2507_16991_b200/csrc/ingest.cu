// ingest.cu — dataset ingestion straight to the device.
//
// Replaces the host-side materialisation of load_dataset (dataset_io.cpp:295-341):
// the reference mmaps node_<type>.<f32|f64>.bin and copies every
// edge_<src>__<rel>__<dst>.u64.bin pair into two host std::vector<Index>
// (dataset_io.cpp:317-326) before building EdgeIndex. Here the file bytes are
// read with pread into two halves of a caller-supplied PINNED staging buffer,
// copied host->device asynchronously while the next half is being read, and
// the interleaved (src, dst) u64 pairs are split into the device int64 src/dst
// arrays by a kernel — the host never holds the COO arrays. Byte lengths are
// validated against the manifest exactly as the reference does
// (MappedFile, dataset_io.cpp:107-119), with the same message text.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <string>

#include "gm_common.cuh"

namespace gm {

__global__ void deinterleave_pairs_kernel(const unsigned long long* __restrict__ pairs, int64_t count,
                                          int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const ulonglong2 p = reinterpret_cast<const ulonglong2*>(pairs)[i];
    src[i] = static_cast<int64_t>(p.x);  // dataset_io.cpp:323-324: static_cast<Index>(u64)
    dst[i] = static_cast<int64_t>(p.y);
  }
}

namespace {

struct File {
  int fd = -1;
  ~File() {
    if (fd >= 0) ::close(fd);
  }
};

gm_status open_checked(const char* path, int64_t expected, File& f) {
  GM_REQUIRE(path, GM_ERR_INVALID_ARGUMENT, "dataset: null path");
  f.fd = ::open(path, O_RDONLY);
  if (f.fd < 0) return fail(GM_ERR_RUNTIME, std::string("dataset: cannot open ") + path);
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) return fail(GM_ERR_RUNTIME, std::string("dataset: cannot stat ") + path);
  if (static_cast<int64_t>(st.st_size) != expected)
    return fail(GM_ERR_RUNTIME, std::string("dataset: ") + path + " holds " + std::to_string(st.st_size) +
                                    " bytes, manifest requires " + std::to_string(expected));
  return GM_OK;
}

gm_status read_fully(int fd, void* buf, size_t bytes, int64_t offset, const char* path) {
  size_t done = 0;
  while (done < bytes) {
    const ssize_t r = ::pread(fd, static_cast<char*>(buf) + done, bytes - done, offset + static_cast<int64_t>(done));
    if (r <= 0) return fail(GM_ERR_RUNTIME, std::string("dataset: short read from ") + path);
    done += static_cast<size_t>(r);
  }
  return GM_OK;
}

struct Events {
  cudaEvent_t e[2] = {nullptr, nullptr};
  ~Events() {
    for (auto& x : e)
      if (x) cudaEventDestroy(x);
  }
};

// Streams `bytes` of the file through the two staging halves; for each chunk
// `consume(dev_or_host_chunk, offset, len, stream)` issues the device work.
template <typename F>
gm_status stream_file(int fd, const char* path, int64_t bytes, void* staging, size_t staging_bytes, size_t align,
                      cudaStream_t st, F&& issue) {
  const size_t half = (staging_bytes / 2) / align * align;
  GM_REQUIRE(half >= align, GM_ERR_INVALID_ARGUMENT, "dataset: staging buffer too small");
  Events ev;
  for (auto& x : ev.e) GM_TRY_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  bool used[2] = {false, false};
  int h = 0;
  for (int64_t off = 0; off < bytes; off += static_cast<int64_t>(half), h ^= 1) {
    const size_t len = static_cast<size_t>(std::min<int64_t>(static_cast<int64_t>(half), bytes - off));
    unsigned char* buf = static_cast<unsigned char*>(staging) + static_cast<size_t>(h) * half;
    if (used[h]) GM_TRY_CUDA(cudaEventSynchronize(ev.e[h]));  // the copy out of this half is done
    gm_status s = read_fully(fd, buf, len, off, path);
    if (s != GM_OK) return s;
    s = issue(buf, off, len, h);
    if (s != GM_OK) return s;
    GM_TRY_CUDA(cudaEventRecord(ev.e[h], st));
    used[h] = true;
  }
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  return GM_OK;
}

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" {

GM_API gm_status gm_read_file_to_device(const char* path, int64_t expected_bytes, void* dst, void* staging,
                                        size_t staging_bytes, gm_stream_t stream) {
  GM_REQUIRE(expected_bytes >= 0, GM_ERR_INVALID_ARGUMENT, "dataset: negative byte count");
  File f;
  gm_status s = open_checked(path, expected_bytes, f);
  if (s != GM_OK) return s;
  if (expected_bytes == 0) return GM_OK;
  GM_REQUIRE(dst && staging, GM_ERR_INVALID_ARGUMENT, "dataset: null buffer");
  cudaStream_t st = as_stream(stream);
  return stream_file(f.fd, path, expected_bytes, staging, staging_bytes, 16, st,
                     [&](const void* buf, int64_t off, size_t len, int) -> gm_status {
                       GM_TRY_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(dst) + off, buf, len,
                                                   cudaMemcpyHostToDevice, st));
                       return GM_OK;
                     });
}

GM_API size_t gm_read_edge_pairs_workspace(size_t staging_bytes) { return staging_bytes / 2 / 16 * 16 * 2; }

GM_API gm_status gm_read_edge_pairs_to_device(const char* path, int64_t edge_count, int64_t* src, int64_t* dst,
                                              void* staging, size_t staging_bytes, void* workspace,
                                              size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(edge_count >= 0, GM_ERR_INVALID_ARGUMENT, "dataset: negative edge count");
  File f;
  const int64_t bytes = edge_count * 16;
  gm_status s = open_checked(path, bytes, f);
  if (s != GM_OK) return s;
  if (edge_count == 0) return GM_OK;
  GM_REQUIRE(src && dst && staging && workspace, GM_ERR_INVALID_ARGUMENT, "dataset: null buffer");
  GM_REQUIRE(workspace_bytes >= gm_read_edge_pairs_workspace(staging_bytes), GM_ERR_INVALID_ARGUMENT,
             "dataset: edge-pair workspace too small");
  cudaStream_t st = as_stream(stream);
  const size_t half = staging_bytes / 2 / 16 * 16;
  return stream_file(f.fd, path, bytes, staging, staging_bytes, 16, st,
                     [&](const void* buf, int64_t off, size_t len, int h) -> gm_status {
                       unsigned char* dev = static_cast<unsigned char*>(workspace) + static_cast<size_t>(h) * half;
                       GM_TRY_CUDA(cudaMemcpyAsync(dev, buf, len, cudaMemcpyHostToDevice, st));
                       const int64_t first = off / 16, n = static_cast<int64_t>(len / 16);
                       const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8));
                       deinterleave_pairs_kernel<<<grid, 256, 0, st>>>(
                           reinterpret_cast<const unsigned long long*>(dev), n, src + first, dst + first);
                       GM_CHECK_LAUNCH("deinterleave_pairs_kernel");
                       return GM_OK;
                     });
}

}  // extern "C"
