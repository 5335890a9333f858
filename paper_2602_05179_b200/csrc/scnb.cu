// scnb.cu -- SCNB scenario-file ingestion straight into HBM.
//
// Format (reference: proj/include/scendp/io.hpp:44-49, proj/src/io.cpp:276-
// 344): little-endian "SCNB" | u16 version = 1 | u32 rows | u32 cols | u16
// dtype = 1 (u32), then rows*cols u32 values, scenario-major.  The header is
// 16 bytes, so the payload is 16-byte aligned and scenario w's column is the
// byte range [16 + 4*rows*w, 16 + 4*rows*(w+1)): a shard of scenarios is one
// contiguous file range and a prefix of m scenarios is a file prefix.
//
// B200 path: no host ScenarioBatch is materialized.  The shard is streamed in
// chunks of whole 32-scenario tiles: pread() (split over up to 8 host
// threads) fills one of two page-locked staging buffers while the previous
// chunk's H2D copy runs on the context stream; each chunk then lands in device memory either as is (reference
// layout) or through to_tiled_kernel into its tile range of the native layout
// (tile t of the shard depends only on chunk t*32/C, so chunks never overlap).
// The reference's error messages and exception class (runtime_error) are kept.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_host;

namespace scendp_host {
template <typename T>
void launch_to_tiled(scendp_ctx* ctx, const T* src, uint64_t rows, uint64_t count, T* dst);
void launch_to_tiled_u8(scendp_ctx* ctx, const uint8_t* src, uint64_t rows, uint64_t count,
                        uint32_t* dst);
}

namespace {

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__,
              "SCNB payloads are little-endian u32 and are copied verbatim");

constexpr uint16_t kScnbVersion = 1;
constexpr uint16_t kScnbDtypeU32 = 1;
constexpr uint64_t kScnbHeader = 16;
constexpr uint64_t kChunkBytes = 64ull << 20;  // per staging buffer

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

uint16_t le16(const unsigned char* b) { return static_cast<uint16_t>(b[0] | (b[1] << 8)); }
uint32_t le32(const unsigned char* b) {
  return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
         (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
}

// pread of `bytes` at `off` split over up to `threads` host threads (the
// page-cache copy is the bottleneck of the pipeline, not PCIe).
void read_parallel(int fd, void* dst, uint64_t bytes, uint64_t off, const std::string& name,
                   const char* what, int threads);

void read_full(int fd, void* dst, uint64_t bytes, uint64_t off, const std::string& name,
               const char* what) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, std::min<uint64_t>(bytes, 1ull << 30), static_cast<off_t>(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) fail(SCENDP_ERR_RUNTIME, name + ": " + what);
    p += r;
    off += static_cast<uint64_t>(r);
    bytes -= static_cast<uint64_t>(r);
  }
}

void read_parallel(int fd, void* dst, uint64_t bytes, uint64_t off, const std::string& name,
                   const char* what, int threads) {
  constexpr uint64_t kMinPart = 8ull << 20;
  const int parts = static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>(static_cast<uint64_t>(threads), bytes / kMinPart)));
  if (parts == 1) return read_full(fd, dst, bytes, off, name, what);
  const uint64_t per = ((bytes + parts - 1) / parts + 4095) & ~uint64_t{4095};
  parallel_parts(parts, [&](int p) {
    const uint64_t lo = std::min(bytes, per * p), hi = std::min(bytes, per * (p + 1));
    if (lo < hi) read_full(fd, static_cast<char*>(dst) + lo, hi - lo, off + lo, name, what);
  });
}

// Read `n` u32 values at file offset `off` and store them narrowed to bytes
// at dst, over up to `threads` readers, each through a small cache-resident
// block (the page-cache copy then stays in cache; only n bytes are written
// to the page-locked buffer).  Returns false when a value needs more than 8
// bits (the caller then reads the chunk as u32).
bool read_parallel_u8(int fd, uint8_t* dst, uint64_t n, uint64_t off, const std::string& name,
                      const char* what, int threads) {
  constexpr uint64_t kBlock = 64ull << 10;  // values per read (256 KB)
  const int parts = static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>(static_cast<uint64_t>(threads), n / (2ull << 20))));
  const uint64_t per = (n + parts - 1) / parts;
  std::vector<uint32_t> wide(parts, 0u);
  parallel_parts(parts, [&](int p) {
    const uint64_t lo = std::min(n, per * p), hi = std::min(n, per * (p + 1));
    std::vector<uint32_t> blk(kBlock);
    uint32_t acc = 0u;
    for (uint64_t a = lo; a < hi; a += kBlock) {
      const uint64_t c = std::min(kBlock, hi - a);
      read_full(fd, blk.data(), c * 4, off + a * 4, name, what);
      for (uint64_t i = 0; i < c; ++i) {
        acc |= blk[i];
        dst[a + i] = static_cast<uint8_t>(blk[i]);
      }
      if (acc >> 8) break;  // wide: the chunk will be re-read as u32
    }
    wide[p] = acc >> 8;
  });
  for (uint32_t w : wide)
    if (w) return false;
  return true;
}

// Header checks in the reference's order and wording (io.cpp:316-333).
scendp_scnb_header open_and_check(const char* path, Fd& f) {
  if (!path) fail(SCENDP_ERR_INVALID_ARGUMENT, "path is null");
  const std::string name(path);
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) fail(SCENDP_ERR_RUNTIME, "cannot open scenario file: " + name);
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) fail(SCENDP_ERR_RUNTIME, "cannot open scenario file: " + name);
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  unsigned char h[kScnbHeader] = {};
  const ssize_t got = ::pread(f.fd, h, kScnbHeader, 0);
  if (got < 4 || std::memcmp(h, "SCNB", 4) != 0)
    fail(SCENDP_ERR_RUNTIME, name + ": bad scenario file magic");
  if (got >= 6 && le16(h + 4) != kScnbVersion)
    fail(SCENDP_ERR_RUNTIME, name + ": unsupported scenario file version " +
                                 std::to_string(le16(h + 4)));
  if (got < static_cast<ssize_t>(kScnbHeader))
    fail(SCENDP_ERR_RUNTIME, name + ": truncated scenario header");
  const uint16_t dtype = le16(h + 14);
  if (dtype != kScnbDtypeU32)
    fail(SCENDP_ERR_RUNTIME, name + ": unsupported scenario dtype " + std::to_string(dtype));
  scendp_scnb_header hdr{};
  hdr.rows = le32(h + 6);
  hdr.count = le32(h + 10);
  if (size < kScnbHeader + hdr.rows * hdr.count * 4)
    fail(SCENDP_ERR_RUNTIME, name + ": truncated scenario payload");
  return hdr;
}

}  // namespace

extern "C" {

scendp_status scendp_scnb_header_read(const char* path, scendp_scnb_header* hdr) {
  return guard([&] {
    if (!hdr) fail(SCENDP_ERR_INVALID_ARGUMENT, "header output is null");
    Fd f;
    *hdr = open_and_check(path, f);
  });
}

scendp_status scendp_scnb_load(scendp_ctx* ctx, const char* path, uint64_t first,
                               uint64_t count, uint32_t layout, uint32_t* out) {
  NvtxRange nvtx("scendp_scnb_load");
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    if (layout != SCENDP_MEM_DEVICE && layout != SCENDP_MEM_DEVICE_TILED)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "layout must be SCENDP_MEM_DEVICE or DEVICE_TILED");
    Fd f;
    const scendp_scnb_header hdr = open_and_check(path, f);
    if (first > hdr.count || count > hdr.count - first)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario range [" + std::to_string(first) + ", " +
                                            std::to_string(first + count) + ") exceeds the " +
                                            std::to_string(hdr.count) + " scenarios of " + path);
    if (count == 0 || hdr.rows == 0) return;
    if (!out) fail(SCENDP_ERR_INVALID_ARGUMENT, "output is null");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const uint64_t rows = hdr.rows;
    const uint64_t col_bytes = rows * 4;
    // chunk = whole tiles, <= kChunkBytes unless one tile is larger
    uint64_t chunk = std::max<uint64_t>(32, (kChunkBytes / col_bytes) & ~uint64_t{31});
    chunk = std::min(chunk, (count + 31) & ~uint64_t{31});
    const uint64_t stage_bytes = chunk * col_bytes;
    const int readers = static_cast<int>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())));
    char* pin[2] = {static_cast<char*>(ctx->pinned_stage(0, stage_bytes)),
                    static_cast<char*>(ctx->pinned_stage(1, stage_bytes))};
    uint32_t* dstage = layout == SCENDP_MEM_DEVICE_TILED
                           ? static_cast<uint32_t*>(ctx->scratch_get(kScrStaging, stage_bytes))
                           : nullptr;
    cudaEvent_t done[2];
    for (auto& e : done) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bool used[2] = {false, false};
    // tiled output: values below 256 (the usual demands) are narrowed to
    // bytes while read and widened by the tiling kernel (1/4 of the PCIe
    // bytes); the first chunk with a wider value switches to u32
    bool narrow = layout == SCENDP_MEM_DEVICE_TILED;
    try {
      for (uint64_t c0 = 0, j = 0; c0 < count; c0 += chunk, ++j) {
        const uint64_t cn = std::min(chunk, count - c0);
        const int b = static_cast<int>(j & 1);
        if (used[b]) CUDA_CHECK(cudaEventSynchronize(done[b]));  // buffer b drained
        if (narrow) {
          uint8_t* p8 = reinterpret_cast<uint8_t*>(pin[b]);
          if (read_parallel_u8(f.fd, p8, cn * rows, kScnbHeader + (first + c0) * col_bytes, path,
                               "truncated scenario payload", readers)) {
            uint8_t* d8 = reinterpret_cast<uint8_t*>(dstage);
            ctx->copy(d8, p8, cn * rows, cudaMemcpyHostToDevice);
            launch_to_tiled_u8(ctx, d8, rows, cn, out + (c0 / 32) * rows * 32);
            CUDA_CHECK(cudaEventRecord(done[b], ctx->stream));
            used[b] = true;
            continue;
          }
          narrow = false;
        }
        read_parallel(f.fd, pin[b], cn * col_bytes, kScnbHeader + (first + c0) * col_bytes,
                      path, "truncated scenario payload", readers);
        if (layout == SCENDP_MEM_DEVICE) {
          ctx->copy(out + c0 * rows, pin[b], cn * col_bytes, cudaMemcpyHostToDevice);
        } else {
          ctx->copy(dstage, pin[b], cn * col_bytes, cudaMemcpyHostToDevice);
          launch_to_tiled<uint32_t>(ctx, dstage, rows, cn, out + (c0 / 32) * rows * 32);
        }
        CUDA_CHECK(cudaEventRecord(done[b], ctx->stream));
        used[b] = true;
      }
      ctx->sync();
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      for (auto& e : done) cudaEventDestroy(e);
      throw;
    }
    for (auto& e : done) CUDA_CHECK(cudaEventDestroy(e));
  });
}

scendp_status scendp_scnb_write(const char* path, const uint32_t* data, uint64_t rows,
                                uint64_t count) {
  return guard([&] {
    if (!path) fail(SCENDP_ERR_INVALID_ARGUMENT, "path is null");
    if (rows > 0xffffffffull || count > 0xffffffffull)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "SCNB rows and cols are u32");
    if (!data && rows * count) fail(SCENDP_ERR_INVALID_ARGUMENT, "data is null");
    const std::string name(path);
    Fd f;
    f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (f.fd < 0) fail(SCENDP_ERR_RUNTIME, "cannot write scenario file: " + name);
    unsigned char h[kScnbHeader] = {'S', 'C', 'N', 'B'};
    auto put16 = [&](int at, uint16_t v) {
      h[at] = static_cast<unsigned char>(v);
      h[at + 1] = static_cast<unsigned char>(v >> 8);
    };
    auto put32 = [&](int at, uint32_t v) {
      for (int b = 0; b < 4; ++b) h[at + b] = static_cast<unsigned char>(v >> (8 * b));
    };
    put16(4, kScnbVersion);
    put32(6, static_cast<uint32_t>(rows));
    put32(10, static_cast<uint32_t>(count));
    put16(14, kScnbDtypeU32);
    auto write_all = [&](const void* src, uint64_t bytes) {
      const char* p = static_cast<const char*>(src);
      while (bytes) {
        const ssize_t r = ::write(f.fd, p, std::min<uint64_t>(bytes, 1ull << 30));
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) fail(SCENDP_ERR_RUNTIME, "cannot write scenario file: " + name);
        p += r;
        bytes -= static_cast<uint64_t>(r);
      }
    };
    write_all(h, kScnbHeader);
    write_all(data, rows * count * 4);
  });
}

}  // extern "C"
