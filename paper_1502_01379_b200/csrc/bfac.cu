// bfac.cu — the reference's .bfac factor file (storage.py:1-186) read straight
// into a device plan and written back from one, byte-identical.
//
// Layout (little-endian; storage.py:3-17):
//   "BFAC" | version u32 | n u64 | levels u32 | rank u32 | count u32
//   per factor: kind u8 | level u32 | block_count u64
//     per block: row_off u64 | col_off u64 | rows u32 | cols u32 | payload
//   payload: rows*cols complex128 column-major (kind 2: rank f64 weights).
//   Factor order: U^L, G descending, M, H ascending, V^L; blocks in iter_blocks
//   order (factors.py:38-41, 97-112, 168-172).
//
// Every record of one factor has the same size, so a factor section is a
// regular array of records: it is streamed through a pinned buffer to the
// device, where one kernel checks each record header against the geometry and
// transposes the payload into the plan's row-major block layout (and the
// reverse for saving). Header mismatches report the failing byte offset, as
// FormatError does (storage.py:40-45).
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "plan.h"

namespace bfly {

namespace {

constexpr int kKindU = 0, kKindG = 1, kKindM = 2, kKindH = 3, kKindV = 4;

struct SectionGeo {
  int kind;
  uint32_t level;
  uint64_t nblocks;
  uint32_t R, C;        // block shape (middle: rank x rank weights)
  uint64_t G, P;        // transfer: groups, pairs; leaf: nb
  uint32_t nt;          // transfer: row parts (branching) or 1 (merge-only); leaf 1
  bool leaf, middle;
};

// Expected (row_off, col_off) of block b of a section (iter_blocks order).
__host__ __device__ inline void block_offsets(const SectionGeo& s, uint32_t rank, uint32_t m, uint64_t b,
                                              uint64_t* r0, uint64_t* c0) {
  if (s.middle) {
    const uint64_t i = b / m, j = b % m;
    *r0 = (i * m + j) * rank;
    *c0 = (j * m + i) * rank;
  } else if (s.leaf) {
    *r0 = b * s.R;
    *c0 = b * s.C;
  } else {
    // block b = (g, t, p) with p fastest; rows of (g,t,p): ((g nt + t) P + p) R, cols (g P + p) C
    const uint64_t p = b % s.P, gt = b / s.P, t = gt % s.nt, g = gt / s.nt;
    *r0 = ((g * s.nt + t) * s.P + p) * s.R;
    *c0 = (g * s.P + p) * s.C;
  }
}

__device__ inline uint64_t ld_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
__device__ inline uint32_t ld_u32(const unsigned char* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}
__device__ inline void st_u64(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}
__device__ inline void st_u32(unsigned char* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

// records [b0, b0 + nrec) of a section: check headers, transpose payloads into dst.
template <typename E>
__global__ void unpack_records(const unsigned char* __restrict__ rec, uint64_t nrec, uint64_t b0, SectionGeo s,
                               uint32_t rank, uint32_t m, uint64_t rec_bytes, E* __restrict__ dst,
                               unsigned long long* bad) {
  for (uint64_t q = blockIdx.x; q < nrec; q += gridDim.x) {
    const unsigned char* h = rec + q * rec_bytes;
    const uint64_t b = b0 + q;
    if (threadIdx.x == 0) {
      uint64_t r0, c0;
      block_offsets(s, rank, m, b, &r0, &c0);
      if (ld_u64(h) != r0 || ld_u64(h + 8) != c0 || ld_u32(h + 16) != s.R || ld_u32(h + 20) != s.C)
        atomicMin(bad, static_cast<unsigned long long>(b));
    }
    if (s.middle) {
      const double* w = reinterpret_cast<const double*>(h + 24);
      using Rl = typename Cx<E>::R;
      for (uint32_t i = threadIdx.x; i < rank; i += blockDim.x)
        reinterpret_cast<Rl*>(dst)[b * rank + i] = static_cast<Rl>(w[i]);
    } else {
      // records are 8-byte aligned only (24-byte headers): read the payload as doubles
      const double* pay = reinterpret_cast<const double*>(h + 24);
      const uint32_t n = s.R * s.C;
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
        const uint32_t i = x / s.C, j = x % s.C;  // row-major destination element (i, j)
        const uint64_t src = 2 * (static_cast<uint64_t>(j) * s.R + i);  // column-major source
        dst[b * n + x] = Cx<E>::make(static_cast<typename Cx<E>::R>(pay[src]),
                                     static_cast<typename Cx<E>::R>(pay[src + 1]));
      }
    }
  }
}

__global__ void pack_records(unsigned char* __restrict__ rec, uint64_t nrec, uint64_t b0, SectionGeo s, uint32_t rank,
                             uint32_t m, uint64_t rec_bytes, const double2* __restrict__ src) {
  for (uint64_t q = blockIdx.x; q < nrec; q += gridDim.x) {
    unsigned char* h = rec + q * rec_bytes;
    const uint64_t b = b0 + q;
    if (threadIdx.x == 0) {
      uint64_t r0, c0;
      block_offsets(s, rank, m, b, &r0, &c0);
      st_u64(h, r0);
      st_u64(h + 8, c0);
      st_u32(h + 16, s.R);
      st_u32(h + 20, s.C);
    }
    if (s.middle) {
      double* w = reinterpret_cast<double*>(h + 24);
      const double* sw = reinterpret_cast<const double*>(src);
      for (uint32_t i = threadIdx.x; i < rank; i += blockDim.x) w[i] = sw[b * rank + i];
    } else {
      double* pay = reinterpret_cast<double*>(h + 24);
      const uint32_t n = s.R * s.C;
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
        const uint32_t j = x / s.R, i = x % s.R;  // column-major destination element (i, j)
        const double2 v = src[b * n + static_cast<uint64_t>(i) * s.C + j];
        pay[2 * x] = v.x;
        pay[2 * x + 1] = v.y;
      }
    }
  }
}

std::vector<SectionGeo> file_sections(const Plan& p) {
  std::vector<SectionGeo> out;
  SectionGeo leaf{};
  leaf.leaf = true;
  leaf.nblocks = p.leaf_nb;
  leaf.R = p.leaf_n0;
  leaf.C = p.rank;
  leaf.nt = 1;
  leaf.level = p.levels;
  auto transfer = [&](int kind, uint32_t i) {
    SectionGeo s{};
    s.kind = kind;
    s.level = p.lev[i].level;
    s.nblocks = p.lev[i].nblocks;
    s.R = p.rank;
    s.C = p.branch * p.rank;
    s.G = p.lev[i].G;
    s.P = p.lev[i].P;
    s.nt = p.lev[i].splits ? p.branch : 1;
    return s;
  };
  SectionGeo u = leaf;
  u.kind = kKindU;
  out.push_back(u);
  for (int i = static_cast<int>(p.nlev) - 1; i >= 0; --i) out.push_back(transfer(kKindG, i));
  SectionGeo mid{};
  mid.kind = kKindM;
  mid.middle = true;
  mid.level = p.half;
  mid.nblocks = static_cast<uint64_t>(p.m) * p.m;
  mid.R = mid.C = p.rank;
  out.push_back(mid);
  for (uint32_t i = 0; i < p.nlev; ++i) out.push_back(transfer(kKindH, i));
  SectionGeo v = leaf;
  v.kind = kKindV;
  out.push_back(v);
  return out;
}

void* section_ptr(const Plan& p, const SectionGeo& s) {
  switch (s.kind) {
    case kKindU: return p.u_leaf;
    case kKindV: return p.v_leaf;
    case kKindM: return p.weights;
    case kKindG: return p.g_lev[s.level - p.half];
    default: return p.h_lev[s.level - p.half];
  }
}

uint64_t record_bytes(const SectionGeo& s, uint32_t rank) {
  return 24 + (s.middle ? 8ull * rank : 16ull * s.R * s.C);
}

struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) fclose(f);
  }
};

int fmt_error(const std::string& msg, uint64_t offset) {
  return fail(BF_EFORMAT, msg + " (at byte " + std::to_string(offset) + ")");
}

}  // namespace

}  // namespace bfly

using namespace bfly;

extern "C" {

int bf_plan_load_bfac(bf_plan** out, const char* path, int dtype, int device) {
  if (!out || !path) return fail(BF_EINVAL, "null argument");
  *out = nullptr;
  FileCloser fc{fopen(path, "rb")};
  if (!fc.f) return fail(BF_EINVAL, std::string("cannot open ") + path);
  unsigned char hdr[28];
  uint64_t off = 0;
  const size_t got = fread(hdr, 1, 28, fc.f);
  if (got < 4 || std::memcmp(hdr, "BFAC", 4) != 0) return fmt_error("bad magic", 0);
  if (got < 28) return fmt_error("truncated: wanted 24 bytes, file ends", 4);
  uint32_t version, levels, rank, count;
  uint64_t n;
  std::memcpy(&version, hdr + 4, 4);
  std::memcpy(&n, hdr + 8, 8);
  std::memcpy(&levels, hdr + 16, 4);
  std::memcpy(&rank, hdr + 20, 4);
  std::memcpy(&count, hdr + 24, 4);
  if (version != 1) return fmt_error("unsupported version " + std::to_string(version), 4);
  off = 28;
  bf_plan* plan = nullptr;
  int rc = bf_plan_create(&plan, n, levels, rank, 1, dtype, device);
  if (rc) return rc;
  Plan& p = plan->p;
  const std::vector<SectionGeo> secs = file_sections(p);
  if (count != secs.size()) {
    bf_plan_destroy(plan);
    return fmt_error("factor count " + std::to_string(count) + " does not match geometry", 24);
  }
  // storage (bf_plan_upload carves it; reuse that path with null sources is not possible, so allocate here)
  {
    const uint64_t es = p.elem(), rs = p.real();
    const uint64_t leaf_elems = p.leaf_nb * p.leaf_n0 * p.rank;
    const uint64_t w_elems = static_cast<uint64_t>(p.m) * p.m * p.rank;
    auto up = [](uint64_t x) { return (x + 255) / 256 * 256; };
    uint64_t bytes = 2 * up(leaf_elems * es) + up(w_elems * rs);
    for (const LevelGeo& g : p.lev) bytes += 2 * up(g.nblocks * p.rank * p.branch * p.rank * es);
    DeviceGuardScope dg(p.device);
    cudaError_t e = cudaMalloc(&p.base, bytes);
    if (e != cudaSuccess) {
      p.base = nullptr;
      bf_plan_destroy(plan);
      return cuda_fail(e, "cudaMalloc(factor storage)");
    }
    p.base_bytes = bytes;
    char* cur = static_cast<char*>(p.base);
    auto carve = [&](uint64_t b) {
      void* r = cur;
      cur += up(b);
      return r;
    };
    p.u_leaf = carve(leaf_elems * es);
    p.v_leaf = carve(leaf_elems * es);
    p.weights = carve(w_elems * rs);
    p.g_lev.assign(p.nlev, nullptr);
    p.h_lev.assign(p.nlev, nullptr);
    for (uint32_t i = 0; i < p.nlev; ++i) p.g_lev[i] = carve(p.lev[i].nblocks * p.rank * p.branch * p.rank * es);
    for (uint32_t i = 0; i < p.nlev; ++i) p.h_lev[i] = carve(p.lev[i].nblocks * p.rank * p.branch * p.rank * es);
  }
  DeviceGuardScope dg(p.device);
  const uint64_t chunk_bytes = 256ull << 20;
  unsigned char* host = nullptr;
  unsigned char* dev = nullptr;
  unsigned long long* bad = nullptr;
  auto cleanup = [&](int code) {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    if (bad) cudaFree(bad);
    if (code) bf_plan_destroy(plan);
    return code;
  };
  if (cudaMallocHost(&host, chunk_bytes) != cudaSuccess || cudaMalloc(&dev, chunk_bytes) != cudaSuccess ||
      cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess)
    return cleanup(fail(BF_ENOMEM, "staging allocation failed"));
  for (const SectionGeo& s : secs) {
    unsigned char fh[13];
    if (fread(fh, 1, 13, fc.f) != 13) return cleanup(fmt_error("truncated: wanted 13 bytes, file ends", off));
    const int kind = fh[0];
    uint32_t level;
    uint64_t declared;
    std::memcpy(&level, fh + 1, 4);
    std::memcpy(&declared, fh + 5, 8);
    if (kind != s.kind || level != s.level)
      return cleanup(fmt_error("unexpected factor kind " + std::to_string(kind) + " level " + std::to_string(level),
                               off));
    off += 13;
    if (declared != s.nblocks)
      return cleanup(fmt_error("factor kind " + std::to_string(kind) + " declares " + std::to_string(declared) +
                                   " blocks, geometry implies " + std::to_string(s.nblocks),
                               off));
    const uint64_t rb = record_bytes(s, rank);
    if (rb > chunk_bytes) return cleanup(fail(BF_EINVAL, "block record larger than the staging buffer"));
    const uint64_t per_chunk = chunk_bytes / rb;
    unsigned long long none = ~0ull;
    if (cudaMemcpy(bad, &none, sizeof(none), cudaMemcpyHostToDevice) != cudaSuccess)
      return cleanup(cuda_fail(cudaGetLastError(), "cudaMemcpy"));
    void* dst = section_ptr(p, s);
    for (uint64_t b0 = 0; b0 < s.nblocks; b0 += per_chunk) {
      const uint64_t nrec = std::min<uint64_t>(per_chunk, s.nblocks - b0);
      const size_t want = nrec * rb;
      const size_t have = fread(host, 1, want, fc.f);
      if (have != want)
        return cleanup(fmt_error("truncated: wanted " + std::to_string(rb) + " bytes, file ends",
                                 off + (have / rb) * rb));
      cudaError_t e = cudaMemcpy(dev, host, want, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "H2D .bfac records"));
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nrec, 148ull * 16));
      if (p.dtype == BF_C128)
        unpack_records<double2><<<grid, 128>>>(dev, nrec, b0, s, rank, p.m, rb, static_cast<double2*>(dst), bad);
      else
        unpack_records<float2><<<grid, 128>>>(dev, nrec, b0, s, rank, p.m, rb, static_cast<float2*>(dst), bad);
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "unpack .bfac records"));
      off += want;
    }
    unsigned long long first_bad = 0;
    cudaMemcpy(&first_bad, bad, sizeof(first_bad), cudaMemcpyDeviceToHost);
    if (first_bad != ~0ull) {
      uint64_t r0, c0;
      block_offsets(s, rank, p.m, first_bad, &r0, &c0);
      const uint64_t at = off - s.nblocks * rb + first_bad * rb + 24;
      return cleanup(fmt_error("block header mismatch: expected (" + std::to_string(r0) + ", " + std::to_string(c0) +
                                   ") (" + std::to_string(s.R) + ", " + std::to_string(s.C) + ")",
                               at));
    }
  }
  unsigned char extra;
  if (fread(&extra, 1, 1, fc.f) == 1) return cleanup(fmt_error("trailing bytes after last factor", off));
  p.uploaded = true;
  if (int frc = plan_fold_leaves(p, nullptr)) return cleanup(frc);
  cleanup(0);
  *out = plan;
  return BF_OK;
}

int bf_plan_save_bfac(const bf_plan* plan, const char* path) {
  if (!plan || !path) return fail(BF_EINVAL, "null argument");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors");
  if (p.dtype != BF_C128 || p.nparts != 1) return fail(BF_EINVAL, "only unsharded complex128 plans are saved");
  // the .bfac header (storage.py:65-93) has no branching field: a quadtree chain saved
  // there would load back as a binary one and fail its block counts
  if (p.branch != 2) return fail(BF_EINVAL, ".bfac holds binary-tree chains only (quadtree plan)");
  FileCloser fc{fopen(path, "wb")};
  if (!fc.f) return fail(BF_EINVAL, std::string("cannot create ") + path);
  DeviceGuardScope dg(p.device);
  const std::vector<SectionGeo> secs = file_sections(p);
  unsigned char hdr[28];
  std::memcpy(hdr, "BFAC", 4);
  const uint32_t version = 1, count = static_cast<uint32_t>(secs.size());
  std::memcpy(hdr + 4, &version, 4);
  std::memcpy(hdr + 8, &p.n, 8);
  std::memcpy(hdr + 16, &p.levels, 4);
  std::memcpy(hdr + 20, &p.rank, 4);
  std::memcpy(hdr + 24, &count, 4);
  if (fwrite(hdr, 1, 28, fc.f) != 28) return fail(BF_ECUDA, "write failed");
  const uint64_t chunk_bytes = 256ull << 20;
  unsigned char* host = nullptr;
  unsigned char* dev = nullptr;
  auto cleanup = [&](int code) {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    return code;
  };
  if (cudaMallocHost(&host, chunk_bytes) != cudaSuccess || cudaMalloc(&dev, chunk_bytes) != cudaSuccess)
    return cleanup(fail(BF_ENOMEM, "staging allocation failed"));
  for (const SectionGeo& s : secs) {
    unsigned char fh[13];
    fh[0] = static_cast<unsigned char>(s.kind);
    std::memcpy(fh + 1, &s.level, 4);
    std::memcpy(fh + 5, &s.nblocks, 8);
    if (fwrite(fh, 1, 13, fc.f) != 13) return cleanup(fail(BF_ECUDA, "write failed"));
    const uint64_t rb = record_bytes(s, p.rank);
    const uint64_t per_chunk = chunk_bytes / rb;
    const double2* src = static_cast<const double2*>(section_ptr(p, s));
    for (uint64_t b0 = 0; b0 < s.nblocks; b0 += per_chunk) {
      const uint64_t nrec = std::min<uint64_t>(per_chunk, s.nblocks - b0);
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nrec, 148ull * 16));
      pack_records<<<grid, 128>>>(dev, nrec, b0, s, p.rank, p.m, rb, src);
      cudaError_t e = cudaMemcpy(host, dev, nrec * rb, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "D2H .bfac records"));
      if (fwrite(host, 1, nrec * rb, fc.f) != nrec * rb) return cleanup(fail(BF_ECUDA, "write failed"));
    }
  }
  return cleanup(BF_OK);
}

int bf_plan_export(const bf_plan* plan, int which, uint32_t level, void* dst, uint64_t dst_bytes, void* stream) {
  if (!plan || !dst) return fail(BF_EINVAL, "null argument");
  const Plan& p = plan->p;
  if (!p.uploaded) return fail(BF_ESTATE, "plan has no factors");
  uint64_t bytes = 0;
  const void* src = nullptr;
  const uint64_t es = p.elem();
  if (which == BF_FACTOR_U || which == BF_FACTOR_V) {
    src = which == BF_FACTOR_U ? p.u_leaf : p.v_leaf;
    bytes = p.leaf_nb * p.leaf_n0 * p.rank * es;
  } else if (which == BF_FACTOR_M) {
    src = p.weights;
    bytes = static_cast<uint64_t>(p.m) * p.m * p.rank * p.real();
  } else if (which == BF_FACTOR_G || which == BF_FACTOR_H) {
    if (level < p.half || level >= p.levels) return fail(BF_EINVAL, "transfer level outside [half, levels)");
    const uint32_t i = level - p.half;
    src = which == BF_FACTOR_G ? p.g_lev[i] : p.h_lev[i];
    bytes = p.lev[i].nblocks * p.rank * p.branch * p.rank * es;
  } else {
    return fail(BF_EINVAL, "unknown factor selector");
  }
  if (dst_bytes < bytes) return fail(BF_EINVAL, "export buffer too small");
  DeviceGuardScope dg(p.device);
  BF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return BF_OK;
}

}  // extern "C"
