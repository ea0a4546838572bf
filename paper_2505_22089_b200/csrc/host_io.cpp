// host_io.cpp -- the data formats either side of the matching path (SURVEY
// §8f rows f2 / f3), native so the host side never parses floats one by one:
//   * feature files ("BMF1", read_features features.cpp:222-249, little-endian
//     primitives binary_io.hpp): header checked like the reference, then the
//     528-byte records (4 keypoint floats + 128 descriptor floats) are read
//     with pread in large blocks by several threads, straight into the
//     caller's buffers (pinned host memory for the H2D path), de-interleaved
//     on the fly;
//   * match files ("BMMT", write_matches_binary hashmatch.cpp:311-332): pairs
//     in IdPair order, stage byte, count, (u32 qi, u32 ti) per match, written
//     from the result's pinned log with one buffered write per block.
// Errors carry the reference's codes and messages (FormatError /
// TruncatedFile, binary_io.hpp:37-67).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <bit>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bandmatch_gpu.h"

static_assert(std::endian::native == std::endian::little, "the file formats are little-endian");

namespace bmg {

void set_last_error(const std::string& msg);

namespace {

constexpr char kFeatMagic[4] = {'B', 'M', 'F', '1'};  // features.cpp:22
constexpr uint32_t kFeatVersion = 1;                  // features.cpp:23
constexpr char kMatchMagic[4] = {'B', 'M', 'M', 'T'}; // hashmatch.cpp:16
constexpr uint32_t kMatchVersion = 1;                 // hashmatch.cpp:17
constexpr size_t kHeader = 24;                        // magic, u32 version, u64 id, u32 count, u32 dim
constexpr size_t kRecord = (4 + BMG_DIM) * sizeof(float);

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

int format_error(const std::string& msg) {
  set_last_error(msg);
  return BMG_FORMAT_ERROR;
}
int truncated(const std::string& what) {
  set_last_error("unexpected end of file while reading " + what);
  return BMG_TRUNCATED_FILE;
}

// header checks in the reference's order (features.cpp:226-236)
int read_header(int fd, const std::string& path, uint64_t* id, uint32_t* count) {
  unsigned char h[kHeader];
  const ssize_t got = pread(fd, h, kHeader, 0);
  const size_t have = got < 0 ? 0 : static_cast<size_t>(got);
  if (have < 4) return truncated("feature file magic");
  if (std::memcmp(h, kFeatMagic, 4) != 0) return format_error("feature file: bad magic, expected \"BMF1\"");
  if (have < 8) return truncated("version");
  uint32_t version, dim;
  std::memcpy(&version, h + 4, 4);
  if (version != kFeatVersion) return format_error("unsupported feature file version " + std::to_string(version));
  if (have < 16) return truncated("image id");
  std::memcpy(id, h + 8, 8);
  if (have < 20) return truncated("feature count");
  std::memcpy(count, h + 16, 4);
  if (have < 24) return truncated("descriptor dim");
  std::memcpy(&dim, h + 20, 4);
  if (dim != BMG_DIM) return format_error("descriptor dim " + std::to_string(dim) + " != 128");
  (void)path;
  return BMG_OK;
}

}  // namespace
}  // namespace bmg

using namespace bmg;

extern "C" {

int bmg_read_features_header(const char* path, uint64_t* image_id, uint64_t* count) {
  if (!path || !image_id || !count) {
    set_last_error("null argument");
    return BMG_INVALID_ARGUMENT;
  }
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return format_error(std::string("cannot open ") + path + " for reading");
  uint32_t n = 0;
  const int rc = read_header(f.fd, path, image_id, &n);
  *count = n;
  return rc;
}

int bmg_read_features(const char* path, uint64_t capacity, float* descriptors_out,
                      float* keypoints_out, int threads, uint64_t* image_id, uint64_t* count) {
  if (!path || !descriptors_out || !image_id || !count) {
    set_last_error("null argument");
    return BMG_INVALID_ARGUMENT;
  }
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return format_error(std::string("cannot open ") + path + " for reading");
  uint32_t n = 0;
  if (const int rc = read_header(f.fd, path, image_id, &n); rc != BMG_OK) return rc;
  *count = n;
  if (n > capacity) {
    set_last_error("feature file holds " + std::to_string(n) + " features, buffer " +
                   std::to_string(capacity));
    return BMG_INVALID_ARGUMENT;
  }
  // a file shorter than its header says fails like the reference's reader,
  // which stops in the keypoint or descriptor field the data ends in
  // (features.cpp:240-246)
  struct stat st{};
  if (fstat(f.fd, &st) != 0) return format_error(std::string("cannot stat ") + path);
  const uint64_t body = static_cast<uint64_t>(st.st_size) > kHeader ? static_cast<uint64_t>(st.st_size) - kHeader : 0;
  if (body < static_cast<uint64_t>(n) * kRecord) return truncated(body % kRecord < 16 ? "keypoint" : "descriptor");
  // blocks of whole records, read and de-interleaved by `threads` workers
  constexpr size_t kBlockRecords = 4096;  // ~2 MiB per read
  const size_t n_blocks = (n + kBlockRecords - 1) / kBlockRecords;
  const int T = static_cast<int>(std::clamp<size_t>(threads > 0 ? threads : 1, 1, std::max<size_t>(n_blocks, 1)));
  std::atomic<size_t> next{0};
  std::atomic<int> status{BMG_OK};
  auto worker = [&] {
    std::vector<unsigned char> buf(kBlockRecords * kRecord);
    for (size_t b; (b = next++) < n_blocks && status.load() == BMG_OK;) {
      const size_t r0 = b * kBlockRecords, nr = std::min<size_t>(kBlockRecords, n - r0);
      const off_t off = static_cast<off_t>(kHeader + r0 * kRecord);
      const ssize_t got = pread(f.fd, buf.data(), nr * kRecord, off);
      size_t have = got < 0 ? 0 : static_cast<size_t>(got);
      while (have < nr * kRecord) {  // pread may return short before EOF
        const ssize_t more = pread(f.fd, buf.data() + have, nr * kRecord - have, off + static_cast<off_t>(have));
        if (more <= 0) break;
        have += static_cast<size_t>(more);
      }
      const size_t full = have / kRecord;
      for (size_t i = 0; i < full; ++i) {
        const unsigned char* rec = buf.data() + i * kRecord;
        if (keypoints_out) std::memcpy(keypoints_out + (r0 + i) * 4, rec, 16);
        std::memcpy(descriptors_out + (r0 + i) * BMG_DIM, rec + 16, BMG_DIM * sizeof(float));
      }
      if (full < nr) status.store(BMG_TRUNCATED_FILE);  // shrank while being read
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (status.load() != BMG_OK) return truncated("descriptor");
  return BMG_OK;
}

int bmg_write_matches_binary(const char* path, uint64_t n_pairs, const uint64_t* pair_ids,
                             const uint64_t* ranges, const int32_t* log, const uint8_t* stages) {
  if (!path || (n_pairs && (!pair_ids || !ranges))) {
    set_last_error("null argument");
    return BMG_INVALID_ARGUMENT;
  }
  for (uint64_t p = 1; p < n_pairs; ++p) {
    const bool ordered = pair_ids[2 * p - 2] < pair_ids[2 * p] ||
                         (pair_ids[2 * p - 2] == pair_ids[2 * p] && pair_ids[2 * p - 1] <= pair_ids[2 * p + 1]);
    if (!ordered) {
      set_last_error("pairs must be sorted by IdPair (sorted_by_pair, hashmatch.cpp:243-250)");
      return BMG_INVALID_ARGUMENT;
    }
  }
  FILE* fp = std::fopen(path, "wb");
  if (!fp) return format_error(std::string("cannot open ") + path + " for writing");
  std::vector<char> big(8u << 20);
  std::setvbuf(fp, big.data(), _IOFBF, big.size());
  bool ok = std::fwrite(kMatchMagic, 1, 4, fp) == 4;
  ok = ok && std::fwrite(&kMatchVersion, 4, 1, fp) == 1;
  ok = ok && std::fwrite(&n_pairs, 8, 1, fp) == 1;
  for (uint64_t p = 0; ok && p < n_pairs; ++p) {
    const uint64_t b = ranges[2 * p], e = ranges[2 * p + 1];
    unsigned char head[21];
    std::memcpy(head, &pair_ids[2 * p], 8);
    std::memcpy(head + 8, &pair_ids[2 * p + 1], 8);
    head[16] = stages ? stages[p] : 0;  // Stage::kInitial unless verified
    const uint32_t cnt = static_cast<uint32_t>(e - b);
    std::memcpy(head + 17, &cnt, 4);
    ok = std::fwrite(head, 1, sizeof(head), fp) == sizeof(head);
    // (qi, ti) int32 pairs are the reference's (u32 qi, u32 ti) records
    if (ok && cnt) ok = std::fwrite(log + 2 * b, 8, cnt, fp) == cnt;
  }
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) return format_error(std::string("write failed for ") + path);
  return BMG_OK;
}

}  // extern "C"
