// slrm_io.cuh — SLRM matrix files streamed straight between disk and HBM.
//
// The reference's on-disk format (matrixio.py:1-27): magic "SLRM", version
// u32 LE, rows u64 LE, cols u64 LE, then the row-major IEEE-754 f64 LE
// payload; reads reject short headers / bad magic / bad version
// (matrixio.py:94-103), short payloads (:104-109) and NaN/Inf (:124-125);
// writes are atomic, temp file + rename (:40-50).  Here a reader never builds
// the m x n float64 matrix on the host: row chunks go disk -> pinned buffer
// (double-buffered, the host reads chunk i+1 while the device copies and
// converts chunk i) -> HBM, converted on the device to the consumer's dtype
// (fp32 X, fp64 X or u8 mask "nonzero = observed", cli.py:165-167) with the
// non-finite count folded into the same pass.  Writers stream the other way;
// spcp_slrm_write_product materialises L = U V^T and S* chunk by chunk
// (solver.py:313-320) so the final decomposition of a problem that only fits
// in HBM reaches disk without an m x n host array.
//
// Included at the end of spcp_api.cu (needs spcp_problem and launch_dense).
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <thread>

namespace spcp {

static constexpr char kSlrmMagic[4] = {'S', 'L', 'R', 'M'};
static constexpr uint32_t kSlrmVersion = 1;
static constexpr size_t kSlrmHeader = 24;  // struct "<4sIQQ"
static constexpr size_t kSlrmChunkBytes = size_t(64) << 20;

// dst[r * ld + c] = convert(src[r * cols + c]); counts non-finite sources.
__global__ void slrm_convert_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                    void* __restrict__ dst, int dtype, int64_t ld,
                                    unsigned long long* __restrict__ nonfinite) {
  const int64_t total = rows * cols;
  unsigned bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double v = __ldg(src + i);
    bad += isfinite(v) ? 0u : 1u;
    const int64_t r = i / cols, c = i - r * cols;
    const int64_t o = r * ld + c;
    if (dtype == SPCP_F32)
      static_cast<float*>(dst)[o] = float(v);
    else if (dtype == SPCP_F64)
      static_cast<double*>(dst)[o] = v;
    else
      static_cast<uint8_t*>(dst)[o] = v != 0.0 ? 1 : 0;
  }
  for (int s = 16; s > 0; s >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, s);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, (unsigned long long)bad);
}

// dst (rows x cols, packed f64) = src (rows x cols, stride ld, f32 or f64).
__global__ void slrm_pack_kernel(const void* __restrict__ src, int dtype, int64_t ld,
                                 int64_t rows, int64_t cols, double* __restrict__ dst) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[i] = dtype == SPCP_F32 ? double(static_cast<const float*>(src)[r * ld + c])
                               : static_cast<const double*>(src)[r * ld + c];
  }
}

__global__ void slrm_count_nonzero_kernel(const double* __restrict__ a, int64_t total,
                                          unsigned long long* __restrict__ cnt) {
  unsigned nz = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x)
    nz += a[i] != 0.0 ? 1u : 0u;
  for (int s = 16; s > 0; s >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, s);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(cnt, (unsigned long long)nz);
}

static int io_fail(int err, const std::string& what) {
  const int code = err == ENOENT ? SPCP_ERR_NOT_FOUND : SPCP_ERR_IO;
  return fail(code, what + ": " + std::strerror(err));
}

static int read_fully(int fd, void* buf, size_t bytes, off_t off, size_t* got) {
  size_t done = 0;
  while (done < bytes) {
    const ssize_t r = pread(fd, static_cast<char*>(buf) + done, bytes - done, off + off_t(done));
    if (r < 0) {
      if (errno == EINTR) continue;
      return errno;
    }
    if (r == 0) break;
    done += size_t(r);
  }
  *got = done;
  return 0;
}

static int write_fully(int fd, const void* buf, size_t bytes, off_t off) {
  size_t done = 0;
  while (done < bytes) {
    const ssize_t w =
        pwrite(fd, static_cast<const char*>(buf) + done, bytes - done, off + off_t(done));
    if (w < 0) {
      if (errno == EINTR) continue;
      return errno;
    }
    done += size_t(w);
  }
  return 0;
}

// Page-cache copies run at a few GB/s per thread: large chunk transfers are
// split over up to kIoThreads threads (pread / pwrite at disjoint offsets).
static constexpr int kIoThreads = 4;
static constexpr size_t kIoSplitMin = size_t(8) << 20;

template <typename Fn>
static int par_io(size_t bytes, Fn&& part) {
  const int nt = int(std::min<size_t>(kIoThreads, std::max<size_t>(1, bytes / kIoSplitMin)));
  if (nt == 1) return part(size_t(0), bytes);
  const size_t step = ((bytes + nt - 1) / nt + 4095) & ~size_t(4095);
  std::vector<std::thread> th;
  std::vector<int> rc(nt, 0);
  for (int t = 0; t < nt; ++t) {
    const size_t b0 = std::min(bytes, t * step), b1 = std::min(bytes, b0 + step);
    auto job = [&, t, b0, b1] { rc[t] = b1 > b0 ? part(b0, b1 - b0) : 0; };
    try {
      th.emplace_back(job);
    } catch (...) {  // no thread available: do this part on the calling thread
      job();
    }
  }
  for (auto& x : th) x.join();
  for (int r : rc)
    if (r) return r;
  return 0;
}

// pread of [off, off + bytes) into buf; *got < bytes only at end of file
static int par_read(int fd, void* buf, size_t bytes, off_t off, size_t* got) {
  std::atomic<size_t> total{0};
  const int e = par_io(bytes, [&](size_t b0, size_t n) {
    size_t g = 0;
    const int r = read_fully(fd, static_cast<char*>(buf) + b0, n, off + off_t(b0), &g);
    total += g;
    return r;
  });
  *got = total.load();
  return e;
}

static int par_write(int fd, const void* buf, size_t bytes, off_t off) {
  return par_io(bytes, [&](size_t b0, size_t n) {
    return write_fully(fd, static_cast<const char*>(buf) + b0, n, off + off_t(b0));
  });
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

struct Pinned {
  void* ptr = nullptr;
  ~Pinned() {
    if (ptr) cudaFreeHost(ptr);
  }
};

struct Events {
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Events() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

// header of an open SLRM file; validates it like matrixio.py:94-109
static int slrm_open(const char* path, Fd& f, int64_t* rows, int64_t* cols) {
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return io_fail(errno, std::string(path));
  unsigned char h[kSlrmHeader];
  size_t got = 0;
  if (int e = read_fully(f.fd, h, kSlrmHeader, 0, &got)) return io_fail(e, std::string(path));
  if (got < kSlrmHeader)
    return fail(SPCP_ERR_MALFORMED_HEADER, std::string(path) + ": file shorter than header");
  if (std::memcmp(h, kSlrmMagic, 4) != 0)
    return fail(SPCP_ERR_MALFORMED_HEADER, std::string(path) + ": bad magic");
  uint32_t version;
  uint64_t r, c;
  std::memcpy(&version, h + 4, 4);
  std::memcpy(&r, h + 8, 8);
  std::memcpy(&c, h + 16, 8);
  if (version != kSlrmVersion)
    return fail(SPCP_ERR_MALFORMED_HEADER,
                std::string(path) + ": unsupported version " + std::to_string(version));
  struct stat st;
  if (fstat(f.fd, &st) != 0) return io_fail(errno, std::string(path));
  const unsigned __int128 expect = (unsigned __int128)r * c * 8u;
  const uint64_t have = uint64_t(st.st_size) - kSlrmHeader;
  if (expect > (unsigned __int128)have)
    return fail(SPCP_ERR_TRUNCATED, std::string(path) + ": payload has " + std::to_string(have) +
                                        " bytes, expected " +
                                        std::to_string((unsigned long long)expect));
  *rows = int64_t(r);
  *cols = int64_t(c);
  return SPCP_OK;
}

// atomic writer: temp file in the target's directory, renamed on success
struct AtomicFile {
  std::string path, tmp;
  Fd f;
  bool done = false;
  int open_tmp(const char* target) {
    path = target;
    const size_t slash = path.rfind('/');
    const std::string dir = slash == std::string::npos ? "." : path.substr(0, slash);
    std::vector<char> name(dir.size() + 32);
    std::snprintf(name.data(), name.size(), "%s/.tmp-XXXXXX.part", dir.c_str());
    f.fd = mkstemps(name.data(), 5);
    if (f.fd < 0) return io_fail(errno, path);
    tmp = name.data();
    return SPCP_OK;
  }
  int write_header(int64_t rows, int64_t cols) {
    unsigned char h[kSlrmHeader];
    std::memcpy(h, kSlrmMagic, 4);
    const uint32_t v = kSlrmVersion;
    const uint64_t r = uint64_t(rows), c = uint64_t(cols);
    std::memcpy(h + 4, &v, 4);
    std::memcpy(h + 8, &r, 8);
    std::memcpy(h + 16, &c, 8);
    return put(h, kSlrmHeader);
  }
  off_t pos = 0;
  int put(const void* buf, size_t bytes) {
    if (int e = par_write(f.fd, buf, bytes, pos)) return io_fail(e, tmp);
    pos += off_t(bytes);
    return SPCP_OK;
  }
  int commit() {
    if (close(f.fd) != 0) {
      f.fd = -1;
      return io_fail(errno, tmp);
    }
    f.fd = -1;
    if (rename(tmp.c_str(), path.c_str()) != 0) return io_fail(errno, path);
    done = true;
    return SPCP_OK;
  }
  ~AtomicFile() {
    if (!done && !tmp.empty()) unlink(tmp.c_str());
  }
};

static int slrm_grid(int64_t total) {
  return int(std::min<int64_t>(std::max<int64_t>(1, ceil_div(total, 256)), 148 * 8));
}

}  // namespace spcp

extern "C" {

int spcp_slrm_header(const char* path, int64_t* rows, int64_t* cols) {
  if (!path || !rows || !cols) return fail(SPCP_ERR_VALUE, "null argument");
  Fd f;
  return slrm_open(path, f, rows, cols);
}

int spcp_slrm_read_device(const char* path, int device, int64_t row0, int64_t rows,
                          int64_t col0, int64_t cols, void* dst, int dst_dtype, int64_t ld,
                          void* stream) {
  if (!path || !dst) return fail(SPCP_ERR_VALUE, "null argument");
  if (dst_dtype != SPCP_F32 && dst_dtype != SPCP_F64 && dst_dtype != SPCP_U8)
    return fail(SPCP_ERR_VALUE, "bad destination dtype");
  Fd f;
  int64_t fr, fc;
  if (int rc = slrm_open(path, f, &fr, &fc)) return rc;
  if (rows < 0) rows = fr - row0;
  if (cols < 0) cols = fc - col0;
  if (row0 < 0 || col0 < 0 || rows < 0 || cols < 0 || row0 + rows > fr || col0 + cols > fc)
    return fail(SPCP_ERR_DIMENSION, std::string(path) + ": requested window outside the " +
                                        std::to_string(fr) + "x" + std::to_string(fc) +
                                        " matrix");
  if (ld < cols) return fail(SPCP_ERR_DIMENSION, "ld < cols");
  if (rows == 0 || cols == 0) return SPCP_OK;
  SPCP_CUDA(cudaSetDevice(device));
  posix_fadvise(f.fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool full_rows = col0 == 0 && cols == fc;
  const int64_t chunk = std::max<int64_t>(1, int64_t(kSlrmChunkBytes / (size_t(cols) * 8)));
  const int64_t crows = std::min(chunk, rows);
  const size_t cbytes = size_t(crows) * cols * 8;
  Pinned pin[2];
  Events ev;
  DevBuf stage, counter;
  int rc;
  for (int b = 0; b < 2; ++b) {
    SPCP_CUDA(cudaHostAlloc(&pin[b].ptr, cbytes, cudaHostAllocDefault));
    SPCP_CUDA(cudaEventCreateWithFlags(&ev.ev[b], cudaEventDisableTiming));
  }
  if ((rc = stage.ensure(cbytes))) return rc;
  if ((rc = counter.ensure(sizeof(unsigned long long)))) return rc;
  SPCP_CUDA(cudaMemsetAsync(counter.ptr, 0, sizeof(unsigned long long), st));
  const size_t esz = dst_dtype == SPCP_F32 ? 4 : dst_dtype == SPCP_F64 ? 8 : 1;
  int i = 0;
  for (int64_t r = 0; r < rows; r += crows, ++i) {
    const int b = i & 1;
    const int64_t nr = std::min(crows, rows - r);
    if (i >= 2) SPCP_CUDA(cudaEventSynchronize(ev.ev[b]));  // H2D of chunk i-2 done
    char* hp = static_cast<char*>(pin[b].ptr);
    const off_t base = off_t(kSlrmHeader) + off_t(row0 + r) * off_t(fc) * 8;
    size_t got = 0;
    if (full_rows) {
      const size_t want = size_t(nr) * cols * 8;
      if (int e = par_read(f.fd, hp, want, base, &got)) return io_fail(e, std::string(path));
      if (got != want) return fail(SPCP_ERR_TRUNCATED, std::string(path) + ": short payload");
    } else {
      // one pread per row of the window, rows split over the I/O threads
      const size_t want = size_t(cols) * 8;
      std::atomic<int64_t> short_rows{0};
      const int e = par_io(size_t(nr) * want, [&](size_t b0, size_t n) {
        const int64_t q0 = int64_t(b0 / want), q1 = int64_t((b0 + n + want - 1) / want);
        for (int64_t q = q0; q < std::min(q1, nr); ++q) {
          // a part boundary may split a row: each part reads whole rows whose
          // first byte lies in it
          if (size_t(q) * want < b0) continue;
          size_t g = 0;
          if (int r = read_fully(f.fd, hp + q * want, want,
                                 base + off_t(q) * off_t(fc) * 8 + off_t(col0) * 8, &g))
            return r;
          if (g != want) ++short_rows;
        }
        return 0;
      });
      if (e) return io_fail(e, std::string(path));
      if (short_rows) return fail(SPCP_ERR_TRUNCATED, std::string(path) + ": short payload");
    }
    SPCP_CUDA(cudaMemcpyAsync(stage.ptr, hp, size_t(nr) * cols * 8, cudaMemcpyHostToDevice, st));
    SPCP_CUDA(cudaEventRecord(ev.ev[b], st));
    slrm_convert_kernel<<<slrm_grid(nr * cols), 256, 0, st>>>(
        stage.as<double>(), nr, cols, static_cast<char*>(dst) + size_t(r) * ld * esz, dst_dtype,
        ld, counter.as<unsigned long long>());
    SPCP_CHECK_LAUNCH("slrm_convert_kernel");
  }
  unsigned long long bad = 0;
  SPCP_CUDA(cudaMemcpyAsync(&bad, counter.ptr, sizeof(bad), cudaMemcpyDeviceToHost, st));
  SPCP_CUDA(cudaStreamSynchronize(st));
  if (bad)
    return fail(SPCP_ERR_NONFINITE, std::string(path) + ": matrix contains NaN or Inf entries");
  return SPCP_OK;
}

int spcp_slrm_write_device(const char* path, int device, const void* src, int src_dtype,
                           int64_t rows, int64_t cols, int64_t ld, void* stream) {
  if (!path || (!src && rows * cols > 0)) return fail(SPCP_ERR_VALUE, "null argument");
  if (src_dtype != SPCP_F32 && src_dtype != SPCP_F64)
    return fail(SPCP_ERR_VALUE, "bad source dtype");
  if (rows < 0 || cols < 0 || ld < cols) return fail(SPCP_ERR_DIMENSION, "bad matrix shape");
  SPCP_CUDA(cudaSetDevice(device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  AtomicFile out;
  int rc;
  if ((rc = out.open_tmp(path))) return rc;
  if ((rc = out.write_header(rows, cols))) return rc;
  if (rows > 0 && cols > 0) {
    const int64_t crows =
        std::min(rows, std::max<int64_t>(1, int64_t(kSlrmChunkBytes / (size_t(cols) * 8))));
    const size_t cbytes = size_t(crows) * cols * 8;
    const size_t esz = src_dtype == SPCP_F32 ? 4 : 8;
    Pinned pin[2];
    Events ev;
    DevBuf stage;
    for (int b = 0; b < 2; ++b) {
      SPCP_CUDA(cudaHostAlloc(&pin[b].ptr, cbytes, cudaHostAllocDefault));
      SPCP_CUDA(cudaEventCreateWithFlags(&ev.ev[b], cudaEventDisableTiming));
    }
    if ((rc = stage.ensure(cbytes))) return rc;
    const int64_t nchunks = ceil_div(rows, crows);
    int64_t prev_rows = 0;
    for (int64_t i = 0; i <= nchunks; ++i) {
      const int b = int(i & 1);
      const int64_t r = i * crows;
      const int64_t nr = i < nchunks ? std::min(crows, rows - r) : 0;
      if (nr > 0) {
        slrm_pack_kernel<<<slrm_grid(nr * cols), 256, 0, st>>>(
            static_cast<const char*>(src) + size_t(r) * ld * esz, src_dtype, ld, nr, cols,
            stage.as<double>());
        SPCP_CHECK_LAUNCH("slrm_pack_kernel");
        SPCP_CUDA(cudaMemcpyAsync(pin[b].ptr, stage.ptr, size_t(nr) * cols * 8,
                                  cudaMemcpyDeviceToHost, st));
        SPCP_CUDA(cudaEventRecord(ev.ev[b], st));
      }
      if (i >= 1) {  // write chunk i-1 while the device produces chunk i
        SPCP_CUDA(cudaEventSynchronize(ev.ev[b ^ 1]));
        if ((rc = out.put(pin[b ^ 1].ptr, size_t(prev_rows) * cols * 8))) return rc;
      }
      prev_rows = nr;
    }
  }
  return out.commit();
}

int spcp_slrm_write_product(spcp_problem* p, int64_t k, const double* z, const char* l_path,
                            const char* s_path, int64_t* nnz_s) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (k < 1) return fail(SPCP_ERR_DIMENSION, "k must be >= 1");
  if (!l_path && !s_path && !nnz_s) return SPCP_OK;
  SPCP_CUDA(cudaSetDevice(p->device));
  const int64_t m = p->m, n = p->n;
  const int64_t crows =
      std::min(m, std::max<int64_t>(1, int64_t(kSlrmChunkBytes / (size_t(n) * 8))));
  const size_t cbytes = size_t(crows) * n * 8;
  AtomicFile lf, sf;
  int rc;
  if (l_path && ((rc = lf.open_tmp(l_path)) || (rc = lf.write_header(m, n)))) return rc;
  if (s_path && ((rc = sf.open_tmp(s_path)) || (rc = sf.write_header(m, n)))) return rc;
  const bool want_s = s_path || nnz_s;
  Pinned lpin[2], spin[2];
  Events ev;
  DevBuf stage, counter;
  for (int b = 0; b < 2; ++b) {
    if (l_path) SPCP_CUDA(cudaHostAlloc(&lpin[b].ptr, cbytes, cudaHostAllocDefault));
    if (s_path) SPCP_CUDA(cudaHostAlloc(&spin[b].ptr, cbytes, cudaHostAllocDefault));
    SPCP_CUDA(cudaEventCreateWithFlags(&ev.ev[b], cudaEventDisableTiming));
  }
  if ((rc = stage.ensure(2 * cbytes))) return rc;
  if ((rc = counter.ensure(sizeof(unsigned long long)))) return rc;
  SPCP_CUDA(cudaMemsetAsync(counter.ptr, 0, sizeof(unsigned long long), p->stream));
  double* lo = l_path ? stage.as<double>() : nullptr;
  double* so = want_s ? stage.as<double>() + crows * n : nullptr;
  const int64_t nchunks = ceil_div(m, crows);
  int64_t prev_rows = 0;
  for (int64_t i = 0; i <= nchunks; ++i) {
    const int b = int(i & 1);
    const int64_t r = i * crows;
    const int64_t nr = i < nchunks ? std::min(crows, m - r) : 0;
    if (nr > 0) {
      rc = p->x64.ptr ? launch_dense<double>(p, 0, k, z, r, nr, lo, so, n, nullptr)
                      : launch_dense<float>(p, 0, k, z, r, nr, lo, so, n, nullptr);
      if (rc) return rc;
      if (want_s) {
        slrm_count_nonzero_kernel<<<slrm_grid(nr * n), 256, 0, p->stream>>>(
            so, nr * n, counter.as<unsigned long long>());
        SPCP_CHECK_LAUNCH("slrm_count_nonzero_kernel");
      }
      if (l_path)
        SPCP_CUDA(cudaMemcpyAsync(lpin[b].ptr, lo, size_t(nr) * n * 8, cudaMemcpyDeviceToHost,
                                  p->stream));
      if (s_path)
        SPCP_CUDA(cudaMemcpyAsync(spin[b].ptr, so, size_t(nr) * n * 8, cudaMemcpyDeviceToHost,
                                  p->stream));
      SPCP_CUDA(cudaEventRecord(ev.ev[b], p->stream));
    }
    if (i >= 1) {
      SPCP_CUDA(cudaEventSynchronize(ev.ev[b ^ 1]));
      const size_t bytes = size_t(prev_rows) * n * 8;
      if (l_path && (rc = lf.put(lpin[b ^ 1].ptr, bytes))) return rc;
      if (s_path && (rc = sf.put(spin[b ^ 1].ptr, bytes))) return rc;
    }
    prev_rows = nr;
  }
  unsigned long long nz = 0;
  SPCP_CUDA(cudaMemcpyAsync(&nz, counter.ptr, sizeof(nz), cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  if (nnz_s) *nnz_s = int64_t(nz);
  if (l_path && (rc = lf.commit())) return rc;
  if (s_path && (rc = sf.commit())) return rc;
  return SPCP_OK;
}

}  // extern "C"
