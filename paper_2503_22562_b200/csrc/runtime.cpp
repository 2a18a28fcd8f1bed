// Host runtime of the Niyama hybrid-batch paged-attention library: KV pool and
// block allocator, per-iteration planner (a2), launch wrappers (a3-a6), NCCL
// head all-gather (a7), iteration-time predictor (a8) and slack (a1).
// C ABI: include/niyama.h.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <queue>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.h"
#include "niyama.h"

using namespace niyama;


namespace {

thread_local std::string g_err;

niyama_status fail(niyama_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

}  // namespace

niyama_status niyama::set_error(niyama_status s, const char* msg) { return fail(s, msg); }

namespace {

#define NY_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(NIYAMA_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define NY_NCCL(x)                                                                          \
  do {                                                                                      \
    ncclResult_t r_ = (x);                                                                  \
    if (r_ != ncclSuccess) return fail(NIYAMA_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Seq {
  std::vector<int32_t> blocks;
  int32_t len = 0;
  uint64_t gen = 0;  // creation generation: a released id reused later is a different sequence
};


// Runs the calling thread on `device` for the scope and restores the caller's device
// (the library never leaves the caller's current device changed).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    if (device < 0) return;
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != device) err = cudaSetDevice(device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct niyama_kv {
  niyama_kv_config cfg{};
  int hq = 0, hkv = 0, d = 0, B = 0, elt = 0, g = 0, row_bytes = 0;
  int64_t chunk_bytes = 0;  // one (block, kv head) chunk
  int64_t chunk_stride = 0;  // between consecutive chunks of one of K / V
  int64_t v_offset = 0;      // V's chunk of (block, kv head) = K's + v_offset
  int64_t half_bytes = 0;   // K (or V) of one layer
  bool has_device = false;
  int num_sms = 148;
  uint8_t* pool = nullptr;
  std::set<int32_t> free_;
  std::unordered_map<int64_t, Seq> seqs;
  ncclComm_t comm = nullptr;
  // Plan metadata goes host -> device through a ring of pinned staging buffers;
  // a buffer is reused only after its previous H2D completed (its event), so the
  // host can plan up to kStaging steps ahead of the device.
  static constexpr int kStaging = 8;
  struct Staging {
    void* h = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
    // device buffer uploaded on copy_stream (async_plan): owned by at most one live plan;
    // `released` is recorded on that plan's stream when it is destroyed, and the next
    // upload into the buffer waits for it (kStaging plans later: long complete)
    uint8_t* d = nullptr;
    size_t dcap = 0;
    cudaEvent_t released = nullptr;
    const void* owner = nullptr;
  } stg[kStaging];
  int stg_next = 0;
  // Plan device buffers come from a library-owned stream-ordered pool that never
  // returns memory to the OS (release threshold = max): the per-step
  // allocate/free is then a pointer bump, never a page map.
  cudaMemPool_t mempool = nullptr;
  // Plans are uploaded on this library-owned stream (their buffers come from `mempool`
  // allocated on it), so a plan's H2D overlaps the caller's previous kernels; every
  // use of the plan makes the caller's stream wait for its upload (plan->ready).
  cudaStream_t copy_stream = nullptr;
  int64_t* trace = nullptr;  // niyama_debug_trace
  niyama_tuning tune = default_tuning();  // niyama_kv_set_tuning (explicit; no environment knobs)
  // per-plan upload events (each plan records its own; returned here on destroy)
  std::vector<cudaEvent_t> free_events;
  uint64_t next_gen = 1;  // sequence generations (rollback identity)
};

// Model inputs of a kv for the predictor (predictor.cpp)
void niyama::kv_model(const niyama_kv* kv, KvModel* m) {
  m->hq = kv->hq;
  m->hkv = kv->hkv;
  m->d = kv->d;
  m->elt = kv->elt;
  m->num_sms = kv->num_sms;
  m->tune = kv->tune;
}

struct niyama_plan {
  niyama_kv* kv = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ready = nullptr;  // this plan's own event, recorded right after its upload (either path)
  int32_t slot = -1;            // staging slot whose device buffer holds the plan (-1: pool)
  size_t meta_bytes = 0;        // uploaded part of dbuf (tables, queues, counters): the append prefetches it
  int32_t T = 0, prefill_rows = 0, D = 0, split_len = 0, R = 0;
  int64_t sum_ctx = 0;
  std::vector<int32_t> slot_map;
  std::vector<int32_t> tables;
  struct Prev { int64_t seq; bool existed; int32_t len; uint64_t gen; };
  std::vector<Prev> prev;  // bookkeeping before this plan (niyama_plan_rollback)
  std::vector<PrefillSlice> slices;
  std::vector<DecodeRow> drows;
  std::vector<UnitRec> uq;    // decode queue, one record per (row, split), LPT order
  std::vector<MergeRec> mq;   // merge queue: split rows by the queue position of their last split
  mutable int32_t launches = 0;  // bf16 attention launches issued with this plan (counter epoch)
  std::vector<int32_t> vgrp, velem;  // V^T append groups / element rows
  int32_t n_tiles = 0, n_units = 0, n_merge_rows = 0;  // n_tiles = prefill work items (q tiles)
  int32_t q_tiles = 0;
  int64_t tile_steps = 0;     // sum over prefill tiles of ceil(visible keys / 128)
  int64_t n_setups = 0;       // prefill work items (q tiles x split-K parts)
  int32_t n_split_tiles = 0;  // q tiles with split-K parts > 1
  int64_t split_parts_total = 0;
  int32_t prefill_ctas = 0;   // CTAs of the bf16 launch that take prefill tiles first
  int32_t grid = 0;           // CTAs of the bf16 launch
  std::vector<RowInfo> rows;
  uint8_t* dbuf = nullptr;
  int32_t* d_slot = nullptr;
  int32_t* d_tables = nullptr;
  PrefillSlice* d_slices = nullptr;
  DecodeRow* d_drows = nullptr;
  RowInfo* d_rows = nullptr;
  UnitRec* d_uq = nullptr;
  MergeRec* d_mq = nullptr;
  int32_t* d_counters = nullptr;
  int32_t* d_vgrp = nullptr;
  int32_t* d_velem = nullptr;
  float* d_part_o = nullptr;
  float* d_part_ml = nullptr;
  float* d_ppart_o = nullptr;
  float* d_ppart_ml = nullptr;
  int32_t* d_pcounters = nullptr;
  int32_t* d_work = nullptr;
};

extern "C" const char* niyama_last_error(void) { return g_err.c_str(); }
extern "C" const char* niyama_version(void) { return "niyama-b200 0.1 (sm_100a)"; }

// ================================================================ KV pool
extern "C" niyama_status niyama_kv_create(const niyama_kv_config* cfg, niyama_kv** out) {
  if (!cfg || !out) return fail(NIYAMA_EINVAL, "cfg/out is NULL");
  *out = nullptr;
  const niyama_kv_config& c = *cfg;
  if (c.num_layers < 1) return fail(NIYAMA_EINVAL, "num_layers < 1");
  if (c.num_q_heads < 1 || c.num_kv_heads < 1 || c.num_q_heads % c.num_kv_heads)
    return fail(NIYAMA_EINVAL, "num_q_heads must be a positive multiple of num_kv_heads");
  const int g = c.num_q_heads / c.num_kv_heads;
  if (g > 128 || (g & (g - 1))) return fail(NIYAMA_EUNSUPPORTED, "num_q_heads/num_kv_heads must be a power of two <= 128");
  if (c.world_size < 1 || c.rank < 0 || c.rank >= c.world_size) return fail(NIYAMA_EINVAL, "world_size/rank");
  if (c.num_kv_heads % c.world_size) return fail(NIYAMA_EINVAL, "num_kv_heads must divide by world_size");
  if (c.dtype != NIYAMA_BF16 && c.dtype != NIYAMA_F32) return fail(NIYAMA_EINVAL, "dtype");
  const int elt = c.dtype == NIYAMA_BF16 ? 2 : 4;
  if (c.head_dim < 1 || (c.head_dim * elt) % 128) return fail(NIYAMA_EUNSUPPORTED, "head_dim*elt must be a multiple of 128 bytes");
  if (c.block_size != 16 && c.block_size != 32 && c.block_size != 64 && c.block_size != 128)
    return fail(NIYAMA_EUNSUPPORTED, "block_size must be 16, 32, 64 or 128");
  if (c.num_blocks < 1) return fail(NIYAMA_EINVAL, "num_blocks < 1");
  if (static_cast<int64_t>(c.num_blocks) * c.block_size >= (int64_t(1) << 31))
    return fail(NIYAMA_EINVAL, "num_blocks*block_size must be < 2^31");
  // shapes the kernels are built for (rejected here, not at the first launch)
  if (c.dtype == NIYAMA_BF16 && (c.head_dim != 128 || g > 8))
    return fail(NIYAMA_EUNSUPPORTED, "bf16: the fused kernel is built for head_dim 128 and Hq/Hkv <= 8");
  if (c.dtype == NIYAMA_F32 && (c.head_dim > 128 || g > 8))
    return fail(NIYAMA_EUNSUPPORTED, "f32: head_dim <= 128 and Hq/Hkv <= 8");
  auto* kv = new niyama_kv();
  kv->cfg = c;
  kv->hq = c.num_q_heads / c.world_size;
  kv->hkv = c.num_kv_heads / c.world_size;
  kv->d = c.head_dim;
  kv->B = c.block_size;
  kv->elt = elt;
  kv->g = g;
  kv->row_bytes = c.head_dim * elt;
  kv->chunk_bytes = static_cast<int64_t>(c.block_size) * kv->row_bytes;
  kv->half_bytes = static_cast<int64_t>(c.num_blocks) * kv->hkv * kv->chunk_bytes;
  // bf16: a (block, kv head)'s K chunk and V^T chunk are adjacent ([layer][block][kv head][K|V]),
  // so a decode stage of B = 16 tokens is ONE 8 KB bulk copy.  f32 (config 1): [layer][K|V][block][kv head].
  const bool adjacent = c.dtype == NIYAMA_BF16;
  kv->chunk_stride = adjacent ? 2 * kv->chunk_bytes : kv->chunk_bytes;
  kv->v_offset = adjacent ? kv->chunk_bytes : kv->half_bytes;
  for (int32_t b = 0; b < c.num_blocks; ++b) kv->free_.insert(kv->free_.end(), b);
  if (c.device != NIYAMA_DEVICE_NONE) {
    kv->has_device = true;
    DeviceGuard dg(c.device);
    cudaError_t e = dg.err;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&kv->num_sms, cudaDevAttrMultiProcessorCount, c.device);
    const size_t bytes = static_cast<size_t>(kv->half_bytes) * 2 * c.num_layers;
    if (e == cudaSuccess) e = cudaMalloc(&kv->pool, bytes);
    if (e == cudaSuccess) e = cudaMemset(kv->pool, 0, bytes);  // stale slots stay finite (masked, P = 0)
    for (int i = 0; i < niyama_kv::kStaging && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&kv->stg[i].ev, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&kv->stg[i].released, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = c.device;
      e = cudaMemPoolCreate(&kv->mempool, &props);
      uint64_t keep = ~uint64_t(0);
      if (e == cudaSuccess) e = cudaMemPoolSetAttribute(kv->mempool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&kv->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && c.dtype == NIYAMA_BF16) e = configure_attention_bf16();  // per device (this one)
    if (e != cudaSuccess) {
      for (auto& st : kv->stg) {
        if (st.ev) cudaEventDestroy(st.ev);
        if (st.released) cudaEventDestroy(st.released);
      }
      if (kv->copy_stream) cudaStreamDestroy(kv->copy_stream);
      if (kv->mempool) cudaMemPoolDestroy(kv->mempool);
      if (kv->pool) cudaFree(kv->pool);
      delete kv;
      return fail(NIYAMA_ECUDA, std::string("kv_create: ") + cudaGetErrorString(e));
    }
  }
  *out = kv;
  return NIYAMA_OK;
}

extern "C" void niyama_kv_destroy(niyama_kv* kv) {
  if (!kv) return;
  if (kv->has_device) {
    DeviceGuard dg(kv->cfg.device);
    cudaDeviceSynchronize();
    if (kv->comm) ncclCommDestroy(kv->comm);
    for (cudaEvent_t ev : kv->free_events) cudaEventDestroy(ev);
    if (kv->pool) cudaFree(kv->pool);
    for (auto& st : kv->stg) {
      if (st.h) cudaFreeHost(st.h);
      if (st.ev) cudaEventDestroy(st.ev);
      if (st.released) cudaEventDestroy(st.released);
      if (st.d) cudaFree(st.d);
    }
    if (kv->copy_stream) cudaStreamDestroy(kv->copy_stream);
    if (kv->mempool) cudaMemPoolDestroy(kv->mempool);
  }
  delete kv;
}

extern "C" niyama_status niyama_kv_release(niyama_kv* kv, int64_t seq_id) {
  if (!kv) return fail(NIYAMA_EINVAL, "kv is NULL");
  auto it = kv->seqs.find(seq_id);
  if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "release: unknown seq " + std::to_string(seq_id));
  for (int32_t b : it->second.blocks) kv->free_.insert(b);
  kv->seqs.erase(it);
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_truncate(niyama_kv* kv, int64_t seq_id, int32_t new_len) {
  if (!kv) return fail(NIYAMA_EINVAL, "kv is NULL");
  auto it = kv->seqs.find(seq_id);
  if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "truncate: unknown seq " + std::to_string(seq_id));
  Seq& q = it->second;
  if (new_len < 0 || new_len > q.len) return fail(NIYAMA_EINVAL, "truncate: new_len outside [0, cached length]");
  const size_t keep = static_cast<size_t>(ceil_div(new_len, kv->B));
  for (size_t k = keep; k < q.blocks.size(); ++k) kv->free_.insert(q.blocks[k]);
  q.blocks.resize(keep);
  q.len = new_len;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_block_table(const niyama_kv* kv, int64_t seq_id, int32_t* out, int32_t cap,
                                               int32_t* n) {
  if (!kv || !n) return fail(NIYAMA_EINVAL, "kv/n is NULL");
  auto it = kv->seqs.find(seq_id);
  if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "block_table: unknown seq " + std::to_string(seq_id));
  *n = static_cast<int32_t>(it->second.blocks.size());
  if (out && cap > 0)
    std::memcpy(out, it->second.blocks.data(), sizeof(int32_t) * std::min<size_t>(cap, it->second.blocks.size()));
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_seq_len(const niyama_kv* kv, int64_t seq_id, int32_t* len) {
  if (!kv || !len) return fail(NIYAMA_EINVAL, "kv/len is NULL");
  auto it = kv->seqs.find(seq_id);
  if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "seq_len: unknown seq " + std::to_string(seq_id));
  *len = it->second.len;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_num_free(const niyama_kv* kv, int32_t* n) {
  if (!kv || !n) return fail(NIYAMA_EINVAL, "kv/n is NULL");
  *n = static_cast<int32_t>(kv->free_.size());
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_gather(niyama_kv* kv, int32_t layer, int64_t seq_id, int32_t len, void* k_out,
                                          void* v_out, niyama_stream stream) {
  if (!kv) return fail(NIYAMA_EINVAL, "kv is NULL");
  if (!kv->has_device) return fail(NIYAMA_EUNSUPPORTED, "no device (NIYAMA_DEVICE_NONE)");
  if (layer < 0 || layer >= kv->cfg.num_layers) return fail(NIYAMA_EINVAL, "layer out of range");
  auto it = kv->seqs.find(seq_id);
  if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "gather: unknown seq " + std::to_string(seq_id));
  if (len < 0 || len > it->second.len) return fail(NIYAMA_EINVAL, "gather: len exceeds cached length");
  if (len == 0) return NIYAMA_OK;
  if (!k_out || !v_out) return fail(NIYAMA_EINVAL, "k_out/v_out is NULL");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  const auto& tbl = it->second.blocks;
  int32_t* d_tbl = nullptr;
  NY_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_tbl), tbl.size() * sizeof(int32_t), s));
  NY_CUDA(cudaMemcpyAsync(d_tbl, tbl.data(), tbl.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  const uint8_t* pk = kv->pool + static_cast<int64_t>(layer) * 2 * kv->half_bytes;
  NY_CUDA(launch_gather(pk, pk + kv->v_offset, d_tbl, len, kv->hkv, kv->row_bytes, kv->B, kv->chunk_stride,
                        kv->cfg.dtype == NIYAMA_BF16 ? 1 : 0, static_cast<uint8_t*>(k_out), static_cast<uint8_t*>(v_out),
                        s));
  NY_CUDA(cudaFreeAsync(d_tbl, s));
  NY_CUDA(cudaStreamSynchronize(s));  // the host table must outlive the pageable copy
  return NIYAMA_OK;
}

// ================================================================ planner
namespace {

void plan_cta_split(niyama_plan* pl, const niyama_kv* kv) {
  const CtaSplit r = cta_split(pl->n_tiles, pl->n_units, pl->tile_steps + NIYAMA_TILE_SETUP_STEPS * pl->n_setups,
                               pl->sum_ctx, kv->hkv, kv->d, kv->elt, kv->g, kv->num_sms, kv->tune.decode_path);
  pl->grid = r.grid;
  pl->prefill_ctas = r.prefill_ctas;
  if (kv->tune.prefill_ctas > 0 && pl->n_tiles > 0) pl->prefill_ctas = std::min(kv->tune.prefill_ctas, pl->grid);
}

}  // namespace

extern "C" niyama_status niyama_plan_create(niyama_kv* kv, const niyama_batch_desc* desc, niyama_stream stream,
                                            niyama_plan** out) {
  if (!kv || !desc || !out) return fail(NIYAMA_EINVAL, "kv/desc/out is NULL");
  *out = nullptr;
  const int P = desc->num_prefill, D = desc->num_decode;
  if (P < 0 || D < 0) return fail(NIYAMA_EINVAL, "num_prefill/num_decode < 0");
  if (P > 0 && (!desc->prefill_seq || !desc->prefill_offset || !desc->prefill_len))
    return fail(NIYAMA_EINVAL, "prefill arrays are NULL");
  if (D > 0 && (!desc->decode_seq || !desc->decode_ctx)) return fail(NIYAMA_EINVAL, "decode arrays are NULL");
  {
    std::vector<int64_t> ids(desc->prefill_seq, desc->prefill_seq + (P > 0 ? P : 0));
    if (D > 0) ids.insert(ids.end(), desc->decode_seq, desc->decode_seq + D);
    std::sort(ids.begin(), ids.end());
    const auto dup = std::adjacent_find(ids.begin(), ids.end());
    if (dup != ids.end()) return fail(NIYAMA_EINVAL, "seq " + std::to_string(*dup) + " appears twice in one batch");
  }
  // ---- validate (no side effects)
  std::vector<std::pair<int64_t, int32_t>> new_len;
  new_len.reserve(P + D);
  int64_t T = 0;
  for (int i = 0; i < P; ++i) {
    const int64_t s = desc->prefill_seq[i];
    const int32_t o = desc->prefill_offset[i], c = desc->prefill_len[i];
    if (o < 0 || c < 0) return fail(NIYAMA_EINVAL, "prefill_offset/prefill_len < 0 (slice " + std::to_string(i) + ")");
    if (static_cast<int64_t>(o) + c > std::numeric_limits<int32_t>::max() / 2)
      return fail(NIYAMA_EINVAL, "prefill_offset+prefill_len too large");
    auto it = kv->seqs.find(s);
    const int32_t cur = it == kv->seqs.end() ? 0 : it->second.len;
    if (cur != o)
      return fail(NIYAMA_ESTATE, "seq " + std::to_string(s) + ": cached " + std::to_string(cur) +
                                     " != prefill_offset " + std::to_string(o));
    new_len.emplace_back(s, o + c);
    T += c;
  }
  for (int j = 0; j < D; ++j) {
    const int64_t s = desc->decode_seq[j];
    const int32_t ctx = desc->decode_ctx[j];
    if (ctx < 1) return fail(NIYAMA_EINVAL, "decode_ctx < 1 (decode " + std::to_string(j) + ")");
    auto it = kv->seqs.find(s);
    if (it == kv->seqs.end()) return fail(NIYAMA_ENOSEQ, "decode of unknown seq " + std::to_string(s));
    if (it->second.len != ctx - 1)
      return fail(NIYAMA_ESTATE, "seq " + std::to_string(s) + ": cached " + std::to_string(it->second.len) +
                                     " != decode_ctx-1 " + std::to_string(ctx - 1));
    new_len.emplace_back(s, ctx);
    T += 1;
  }
  if (T > std::numeric_limits<int32_t>::max() / 4) return fail(NIYAMA_EINVAL, "batch too large");
  int64_t need_total = 0;
  for (auto& [s, n] : new_len) {
    auto it = kv->seqs.find(s);
    const int64_t have = it == kv->seqs.end() ? 0 : static_cast<int64_t>(it->second.blocks.size());
    need_total += std::max<int64_t>(0, ceil_div(n, kv->B) - have);
  }
  if (need_total > static_cast<int64_t>(kv->free_.size()))
    return fail(NIYAMA_ENOBLOCKS, "need " + std::to_string(need_total) + " blocks, " +
                                      std::to_string(kv->free_.size()) + " free");
  // the staging buffer this plan will use must have finished its previous H2D
  niyama_kv::Staging* stg = nullptr;
  if (kv->has_device) {
    stg = &kv->stg[kv->stg_next];
    if (stg->pending) {
      NY_CUDA(cudaEventSynchronize(stg->ev));
      stg->pending = false;
    }
  }
  // ---- commit: smallest free ids, descriptor order (R9); remember how to undo it
  struct Undo { int64_t seq; bool existed; size_t nblocks; int32_t len; uint64_t gen; };
  std::vector<Undo> undo;
  undo.reserve(new_len.size());
  for (auto& [s, n] : new_len) {
    auto it = kv->seqs.find(s);
    undo.push_back(it == kv->seqs.end() ? Undo{s, false, 0, 0, 0}
                                        : Undo{s, true, it->second.blocks.size(), it->second.len, it->second.gen});
  }
  auto rollback = [&]() {
    for (auto it = undo.rbegin(); it != undo.rend(); ++it) {
      Seq& q = kv->seqs[it->seq];
      for (size_t k = it->nblocks; k < q.blocks.size(); ++k) kv->free_.insert(q.blocks[k]);
      if (!it->existed) {
        kv->seqs.erase(it->seq);
      } else {
        q.blocks.resize(it->nblocks);
        q.len = it->len;
      }
    }
  };
  for (auto& [s, n] : new_len) {
    Seq& q = kv->seqs[s];
    if (q.gen == 0) q.gen = kv->next_gen++;  // created by this plan
    const int64_t need = std::max<int64_t>(0, ceil_div(n, kv->B) - static_cast<int64_t>(q.blocks.size()));
    for (int64_t k = 0; k < need; ++k) {
      auto fit = kv->free_.begin();
      q.blocks.push_back(*fit);
      kv->free_.erase(fit);
    }
    q.len = n;
  }
  // ---- host metadata
  auto* pl = new niyama_plan();
  pl->kv = kv;
  for (const auto& u : undo)
    pl->prev.push_back(niyama_plan::Prev{u.seq, u.existed, u.len, u.existed ? u.gen : kv->seqs[u.seq].gen});
  pl->stream = reinterpret_cast<cudaStream_t>(stream);
  pl->T = static_cast<int32_t>(T);
  pl->D = D;
  const int B = kv->B, g = kv->g, hkv = kv->hkv;
  std::vector<int32_t> tbl_off(P + D);
  std::vector<Seq*> seq_of(P + D);
  {
    size_t nb = 0;
    for (int k = 0; k < P + D; ++k) {
      seq_of[k] = &kv->seqs[new_len[k].first];
      nb += seq_of[k]->blocks.size();
    }
    pl->tables.reserve(nb + 1);
  }
  for (int k = 0; k < P + D; ++k) {
    const Seq& q = *seq_of[k];
    tbl_off[k] = static_cast<int32_t>(pl->tables.size());
    pl->tables.insert(pl->tables.end(), q.blocks.begin(), q.blocks.end());
  }
  if (pl->tables.empty()) pl->tables.push_back(0);
  pl->slot_map.reserve(T);
  pl->rows.reserve(T);
  std::vector<int32_t> row0(P);
  int32_t row = 0;
  for (int i = 0; i < P; ++i) {
    const Seq& q = *seq_of[i];
    row0[i] = row;
    const int32_t o = desc->prefill_offset[i];
    for (int32_t k = 0; k < desc->prefill_len[i]; ++k, ++row) {
      const int32_t pos = o + k;
      pl->slot_map.push_back(q.blocks[pos / B] * B + pos % B);
      pl->rows.push_back(RowInfo{tbl_off[i], pos + 1});
    }
  }
  pl->prefill_rows = row;
  // V^T append groups (see AppendParams): 8-aligned runs of 8 positions inside a slice
  for (int i = 0; i < P; ++i) {
    const int32_t o = desc->prefill_offset[i], c = desc->prefill_len[i];
    int32_t k = 0;
    while (k < c) {
      const int32_t pos = o + k;
      if ((pos & 7) == 0 && k + 8 <= c) {
        pl->vgrp.push_back(row0[i] + k);
        k += 8;
      } else {
        pl->velem.push_back(row0[i] + k);
        k += 1;
      }
    }
  }
  for (int j = 0; j < D; ++j) pl->velem.push_back(row + j);
  for (int j = 0; j < D; ++j, ++row) {
    const Seq& q = *seq_of[P + j];
    const int32_t pos = desc->decode_ctx[j] - 1;
    pl->slot_map.push_back(q.blocks[pos / B] * B + pos % B);
    pl->rows.push_back(RowInfo{tbl_off[P + j], pos + 1});
    pl->sum_ctx += desc->decode_ctx[j];
  }
  auto tier_of = [&](int k) -> int { return desc->tier ? desc->tier[k] : 0; };
  // prefill slices (a4): 128 MMA rows = g heads x R rows; slices with the most keys first
  pl->R = 128 / g;
  {
    std::vector<int> order;
    for (int i = 0; i < P; ++i)
      if (desc->prefill_len[i] > 0) order.push_back(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const int64_t ka = static_cast<int64_t>(desc->prefill_offset[a]) + desc->prefill_len[a];
      const int64_t kb = static_cast<int64_t>(desc->prefill_offset[b]) + desc->prefill_len[b];
      return ka != kb ? ka > kb : tier_of(a) < tier_of(b);
    });
    int32_t tbase = 0;
    for (int i : order) {
      PrefillSlice sl{};
      sl.tbl = tbl_off[i];
      sl.o = desc->prefill_offset[i];
      sl.c = desc->prefill_len[i];
      sl.row0 = row0[i];
      sl.nqt = static_cast<int32_t>(ceil_div(sl.c, pl->R));
      sl.tbase = tbase;
      sl.parts = 1;
      tbase += sl.nqt * hkv;  // work items = 128-row q tiles (split-K parts are set below)
      for (int32_t qt = 0; qt < sl.nqt; ++qt)
        pl->tile_steps += hkv * ceil_div(static_cast<int64_t>(sl.o) + std::min<int64_t>(sl.c, (qt + 1LL) * pl->R), 128);
      pl->q_tiles += sl.nqt * hkv;
      pl->slices.push_back(sl);
    }
    pl->n_tiles = tbase;
  }
  // decode rows (a5): split [0, ctx) into split_len pieces; longest rows first
  int32_t max_ctx = 0;
  for (int j = 0; j < D; ++j) max_ctx = std::max(max_ctx, desc->decode_ctx[j]);
  pl->split_len = choose_split_len(pl->sum_ctx, max_ctx, hkv, kv->num_sms);
  if (kv->tune.split_len > 0 && ceil_div(max_ctx, kv->tune.split_len) <= 4095) pl->split_len = kv->tune.split_len;
  {
    std::vector<int> order(D);
    for (int j = 0; j < D; ++j) order[j] = j;
    std::sort(order.begin(), order.end(), [&](int a, int b) {  // ties: tier, then descriptor order
      if (desc->decode_ctx[a] != desc->decode_ctx[b]) return desc->decode_ctx[a] > desc->decode_ctx[b];
      if (tier_of(P + a) != tier_of(P + b)) return tier_of(P + a) < tier_of(P + b);
      return a < b;
    });
    // Splits of a row of ctx L (a5): n_full = ceil(L/q) - 1 pieces of q = split_len
    // tokens, then the last piece (1..q tokens) cut into pieces of
    // min(q, max(256, q / tail_div)) tokens (measured: 64-token pieces cost more in
    // partials and merges than they win at the tail; 512-token ones at q = 2048 win
    // 640 -> 613 us on 256 x 4096 decodes).  The queue (LPT) takes every full piece first (longest rows first), then
    // the small pieces longest first, so the final phase of the launch is made of
    // short units and the warps run dry together.  Boundaries depend only on the
    // row's ctx and batch totals (deterministic results).
    const int32_t q = pl->split_len;
    const int32_t small = std::min<int32_t>(q, std::max<int32_t>(kv->tune.tail_min, q / kv->tune.tail_div));
    auto n_full_of = [&](int32_t L) { return static_cast<int32_t>(ceil_div(L, q)) - 1; };
    int32_t ubase = 0;
    pl->drows.reserve(D);
    for (int j : order) {
      DecodeRow r{};
      r.tbl = tbl_off[P + j];
      r.ctx = desc->decode_ctx[j];
      r.row = pl->prefill_rows + j;
      const int32_t nf = n_full_of(r.ctx);
      r.nsplit = nf + static_cast<int32_t>(ceil_div(r.ctx - nf * q, small));
      r.ubase = ubase;
      ubase += r.nsplit * hkv;
      if (r.nsplit > 1) ++pl->n_merge_rows;
      pl->drows.push_back(r);
    }
    // heads of one (row, split) are consecutive queue entries
    auto entry = [&](int32_t r, int32_t sp) {
      const DecodeRow& dr = pl->drows[r];
      const int32_t nf = n_full_of(dr.ctx);
      UnitRec u{};
      u.tbl = dr.tbl;
      u.row = dr.row;
      u.k0 = sp < nf ? sp * q : nf * q + (sp - nf) * small;
      u.k1 = std::min(dr.ctx, sp < nf ? u.k0 + q : u.k0 + small);
      u.nsplit = dr.nsplit;
      u.pbase = dr.ubase + sp * hkv;
      u.phys0 = pl->tables[dr.tbl + u.k0 / B];
      u.phys1 = pl->tables[dr.tbl + std::min(u.k0 + 16, u.k1 - 1) / B];
      u.phys2 = pl->tables[dr.tbl + std::min(u.k0 + 32, u.k1 - 1) / B];
      u.crow = r;
      pl->uq.push_back(u);
    };
    pl->uq.reserve(static_cast<size_t>(ubase / std::max(hkv, 1)) + 1);
    for (int32_t r = 0; r < static_cast<int32_t>(pl->drows.size()); ++r)
      for (int32_t sp = 0; sp < n_full_of(pl->drows[r].ctx); ++sp) entry(r, sp);
    struct Piece {
      int32_t len, r, sp;
    };
    std::vector<Piece> pieces;
    for (int32_t r = 0; r < static_cast<int32_t>(pl->drows.size()); ++r) {
      const DecodeRow& dr = pl->drows[r];
      const int32_t nf = n_full_of(dr.ctx);
      for (int32_t sp = nf; sp < dr.nsplit; ++sp) {
        const int32_t k0 = nf * q + (sp - nf) * small;
        pieces.push_back(Piece{std::min(dr.ctx, k0 + small) - k0, r, sp});
      }
    }
    std::sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) {
      if (a.len != b.len) return a.len > b.len;
      return a.r != b.r ? a.r < b.r : a.sp < b.sp;
    });
    for (const Piece& pc : pieces) entry(pc.r, pc.sp);
    // merge queue (a6): rows with splits, in the order their last split is queued
    std::vector<int32_t> last(pl->drows.size(), -1);
    for (int32_t e = 0; e < static_cast<int32_t>(pl->uq.size()); ++e) last[pl->uq[e].crow] = e;
    std::vector<int32_t> mrows;
    for (int32_t r = 0; r < static_cast<int32_t>(pl->drows.size()); ++r)
      if (pl->drows[r].nsplit > 1) mrows.push_back(r);
    std::sort(mrows.begin(), mrows.end(), [&](int32_t a, int32_t b) { return last[a] < last[b]; });
    for (int32_t r : mrows) {
      const DecodeRow& dr = pl->drows[r];
      pl->mq.push_back(MergeRec{dr.row, dr.ubase, dr.nsplit, r});
    }
    pl->n_units = ubase;
  }
  // prefill split-K (internal.h): parts per slice, work items and their setup cost
  {
    const int32_t target = prefill_parts_target(pl->q_tiles, pl->n_units, pl->tile_steps + NIYAMA_TILE_SETUP_STEPS * pl->q_tiles,
                                                pl->sum_ctx, hkv, kv->d, kv->elt, g, kv->num_sms, kv->tune.decode_path,
                                                kv->tune.prefill_split);
    int32_t tbase = 0, pbase = 0;
    pl->n_setups = 0;
    for (PrefillSlice& sl : pl->slices) {
      const int64_t min_steps = ceil_div(static_cast<int64_t>(sl.o) + std::min<int64_t>(sl.c, pl->R), 128);
      sl.parts = target > 1 ? prefill_parts_of_slice(target, min_steps) : 1;
      sl.tbase = tbase;
      sl.pbase = sl.parts > 1 ? pbase : 0;
      tbase += sl.nqt * hkv * sl.parts;
      if (sl.parts > 1) pbase += sl.nqt * hkv;
      pl->n_setups += static_cast<int64_t>(sl.nqt) * hkv * sl.parts;
      pl->split_parts_total += sl.parts > 1 ? static_cast<int64_t>(sl.nqt) * hkv * sl.parts : 0;
    }
    pl->n_tiles = tbase;
    pl->n_split_tiles = pbase;
  }
  plan_cta_split(pl, kv);
  // ---- device copy: one allocation, one H2D
  if (kv->has_device) {
    const size_t A = 256;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off = align_up(off + std::max<size_t>(bytes, 4), A);
      return o;
    };
    const size_t o_slot = take(pl->slot_map.size() * 4);
    const size_t o_tbl = take(pl->tables.size() * 4);
    const size_t o_tiles = take(pl->slices.size() * sizeof(PrefillSlice));
    const size_t o_units = take(pl->drows.size() * sizeof(DecodeRow));
    const size_t o_rows = take(pl->rows.size() * sizeof(RowInfo));
    const size_t o_uq = take(pl->uq.size() * sizeof(UnitRec));
    const size_t o_mq = take(pl->mq.size() * sizeof(MergeRec));
    const size_t o_vgrp = take(pl->vgrp.size() * 4);
    const size_t o_velem = take(pl->velem.size() * 4);
    const size_t o_work = take(32);  // [8] zero-initialised through the H2D (with the counters)
    const size_t o_cnt = take(pl->drows.size() * static_cast<size_t>(hkv) * 4);
    const size_t o_pcnt = take(static_cast<size_t>(pl->n_split_tiles) * 4);
    const size_t meta_bytes = off;
    pl->meta_bytes = meta_bytes;
    const size_t o_part_o = take(static_cast<size_t>(pl->n_units) * g * kv->d * 4);
    const size_t o_part_ml = take(static_cast<size_t>(pl->n_units) * g * 2 * 4);
    const size_t o_ppart_o = take(static_cast<size_t>(pl->split_parts_total) * 128 * kv->d * 4);
    const size_t o_ppart_ml = take(static_cast<size_t>(pl->split_parts_total) * 128 * 2 * 4);
    const size_t total = off;
    // upload on the library's copy stream into the staging slot's own device buffer when
    // no live plan holds it (the common case); otherwise from the pool on the caller's stream
    const bool use_slot = kv->tune.plan_copy_stream && stg->owner == nullptr;
    cudaStream_t s = use_slot ? kv->copy_stream : pl->stream;  // upload stream
    DeviceGuard dg(kv->cfg.device);
    cudaError_t e = dg.err;
    if (e == cudaSuccess) {  // this plan's own upload event (pooled)
      if (kv->free_events.empty()) {
        e = cudaEventCreateWithFlags(&pl->ready, cudaEventDisableTiming);
      } else {
        pl->ready = kv->free_events.back();
        kv->free_events.pop_back();
      }
    }
    if (e == cudaSuccess && use_slot) {
      if (e == cudaSuccess && stg->dcap < total) {
        if (stg->d) e = cudaFree(stg->d);  // grows rarely (first plans, larger batches)
        stg->d = nullptr;
        stg->dcap = 0;
        const size_t cap = total + total / 4 + (1 << 20);
        if (e == cudaSuccess) e = cudaMalloc(&stg->d, cap);
        if (e == cudaSuccess) stg->dcap = cap;
      }
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, stg->released, 0);  // its previous plan's kernels
      if (e == cudaSuccess) {
        pl->dbuf = stg->d;
        pl->slot = kv->stg_next;
        stg->owner = pl;
      }
    } else if (e == cudaSuccess) {
      e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&pl->dbuf), total, kv->mempool, s);
    }
    if (e == cudaSuccess && stg->cap < meta_bytes) {
      if (stg->h) cudaFreeHost(stg->h);
      stg->h = nullptr;
      stg->cap = 0;
      e = cudaMallocHost(&stg->h, std::max<size_t>(meta_bytes, 1 << 20));
      if (e == cudaSuccess) stg->cap = std::max<size_t>(meta_bytes, 1 << 20);
    }
    if (e == cudaSuccess) {
      uint8_t* h = static_cast<uint8_t*>(stg->h);
      std::memcpy(h + o_slot, pl->slot_map.data(), pl->slot_map.size() * 4);
      std::memcpy(h + o_tbl, pl->tables.data(), pl->tables.size() * 4);
      std::memcpy(h + o_tiles, pl->slices.data(), pl->slices.size() * sizeof(PrefillSlice));
      std::memcpy(h + o_units, pl->drows.data(), pl->drows.size() * sizeof(DecodeRow));
      std::memcpy(h + o_rows, pl->rows.data(), pl->rows.size() * sizeof(RowInfo));
      std::memcpy(h + o_uq, pl->uq.data(), pl->uq.size() * sizeof(UnitRec));
      std::memcpy(h + o_mq, pl->mq.data(), pl->mq.size() * sizeof(MergeRec));
      std::memcpy(h + o_vgrp, pl->vgrp.data(), pl->vgrp.size() * 4);
      std::memcpy(h + o_velem, pl->velem.data(), pl->velem.size() * 4);
      std::memset(h + o_work, 0, meta_bytes - o_work);
      e = cudaMemcpyAsync(pl->dbuf, h, meta_bytes, cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess) e = cudaEventRecord(stg->ev, s);  // staging buffer reusable after this
    if (e == cudaSuccess) e = cudaEventRecord(pl->ready, s);  // every use of the plan waits for this
    if (e != cudaSuccess) {
      rollback();  // the error leaves the pool as it was
      if (pl->ready) kv->free_events.push_back(pl->ready);
      if (pl->slot >= 0)
        stg->owner = nullptr;
      else if (pl->dbuf)
        cudaFreeAsync(pl->dbuf, s);
      delete pl;
      return fail(NIYAMA_ECUDA, std::string("plan_create: ") + cudaGetErrorString(e));
    }
    stg->pending = true;
    kv->stg_next = (kv->stg_next + 1) % niyama_kv::kStaging;
    pl->d_slot = reinterpret_cast<int32_t*>(pl->dbuf + o_slot);
    pl->d_tables = reinterpret_cast<int32_t*>(pl->dbuf + o_tbl);
    pl->d_slices = reinterpret_cast<PrefillSlice*>(pl->dbuf + o_tiles);
    pl->d_drows = reinterpret_cast<DecodeRow*>(pl->dbuf + o_units);
    pl->d_rows = reinterpret_cast<RowInfo*>(pl->dbuf + o_rows);
    pl->d_uq = reinterpret_cast<UnitRec*>(pl->dbuf + o_uq);
    pl->d_mq = reinterpret_cast<MergeRec*>(pl->dbuf + o_mq);
    pl->d_counters = reinterpret_cast<int32_t*>(pl->dbuf + o_cnt);
    pl->d_vgrp = reinterpret_cast<int32_t*>(pl->dbuf + o_vgrp);
    pl->d_velem = reinterpret_cast<int32_t*>(pl->dbuf + o_velem);
    pl->d_part_o = reinterpret_cast<float*>(pl->dbuf + o_part_o);
    pl->d_part_ml = reinterpret_cast<float*>(pl->dbuf + o_part_ml);
    pl->d_pcounters = reinterpret_cast<int32_t*>(pl->dbuf + o_pcnt);
    pl->d_ppart_o = reinterpret_cast<float*>(pl->dbuf + o_ppart_o);
    pl->d_ppart_ml = reinterpret_cast<float*>(pl->dbuf + o_ppart_ml);
    pl->d_work = reinterpret_cast<int32_t*>(pl->dbuf + o_work);
  }
  *out = pl;
  return NIYAMA_OK;
}

extern "C" void niyama_plan_destroy(niyama_plan* plan) {
  if (!plan) return;
  if (plan->ready) plan->kv->free_events.push_back(plan->ready);  // re-recorded by a later plan
  if (plan->dbuf) {
    DeviceGuard dg(plan->kv->cfg.device);
    if (plan->slot >= 0) {  // the slot's buffer may be re-uploaded once this plan's kernels are done
      niyama_kv::Staging& st = plan->kv->stg[plan->slot];
      cudaEventRecord(st.released, plan->stream);
      st.owner = nullptr;
    } else {
      cudaFreeAsync(plan->dbuf, plan->stream);
    }
  }
  delete plan;
}

extern "C" niyama_status niyama_plan_rollback(niyama_kv* kv, niyama_plan* plan) {
  if (!kv || !plan || plan->kv != kv) return fail(NIYAMA_EINVAL, "kv/plan mismatch");
  // An entry applies only to the sequence the plan saw: same id AND same generation (a
  // released id reused by a later plan is another sequence and is left alone).
  auto target = [&](const niyama_plan::Prev& pv) -> Seq* {
    auto sit = kv->seqs.find(pv.seq);
    return sit == kv->seqs.end() || sit->second.gen != pv.gen ? nullptr : &sit->second;
  };
  for (const auto& pv : plan->prev) {  // validate everything before any change
    const Seq* q = target(pv);
    if (q && pv.existed && pv.len > q->len)
      return fail(NIYAMA_ESTATE, "rollback: seq " + std::to_string(pv.seq) + " is shorter than before the plan");
  }
  for (auto it = plan->prev.rbegin(); it != plan->prev.rend(); ++it) {
    Seq* q = target(*it);
    if (!q) continue;  // released (or released and re-created) meanwhile
    if (!it->existed) {
      for (int32_t b : q->blocks) kv->free_.insert(b);
      kv->seqs.erase(it->seq);
      continue;
    }
    const size_t keep = static_cast<size_t>(ceil_div(it->len, kv->B));
    for (size_t k = keep; k < q->blocks.size(); ++k) kv->free_.insert(q->blocks[k]);
    q->blocks.resize(keep);
    q->len = it->len;
  }
  plan->prev.clear();
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_plan_get_info(const niyama_plan* plan, niyama_plan_info* out) {
  if (!plan || !out) return fail(NIYAMA_EINVAL, "plan/out is NULL");
  out->num_rows = plan->T;
  out->num_prefill_rows = plan->prefill_rows;
  out->num_decode = plan->D;
  out->num_prefill_tiles = plan->q_tiles;
  out->num_decode_units = plan->n_units;
  out->split_len = plan->split_len;
  out->rows_per_tile = plan->R;
  out->prefill_ctas = plan->prefill_ctas;
  out->sum_ctx = plan->sum_ctx;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_plan_slots(const niyama_plan* plan, int32_t* block_out, int32_t* slot_out,
                                           int32_t cap) {
  if (!plan || !block_out || !slot_out) return fail(NIYAMA_EINVAL, "plan/block_out/slot_out is NULL");
  const int B = plan->kv->B;
  for (int32_t r = 0; r < plan->T && r < cap; ++r) {
    block_out[r] = plan->slot_map[r] / B;
    slot_out[r] = plan->slot_map[r] % B;
  }
  return NIYAMA_OK;
}

// ================================================================ launches
namespace {
niyama_status check_launch(niyama_kv* kv, const niyama_plan* plan, int32_t layer) {
  if (!kv || !plan) return fail(NIYAMA_EINVAL, "kv/plan is NULL");
  if (plan->kv != kv) return fail(NIYAMA_EINVAL, "plan belongs to another niyama_kv");
  if (!kv->has_device) return fail(NIYAMA_EUNSUPPORTED, "no device (NIYAMA_DEVICE_NONE): there is no CPU path");
  if (layer < 0 || layer >= kv->cfg.num_layers) return fail(NIYAMA_EINVAL, "layer out of range");
  return NIYAMA_OK;
}

// The caller's stream waits for the plan's upload (kv->copy_stream) before using it.
cudaError_t wait_plan(const niyama_plan* plan, niyama_stream stream) {
  if (!plan->ready) return cudaSuccess;
  return cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), plan->ready, 0);
}
}  // namespace

namespace {
niyama_status fill_append(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* k_new, const void* v_new,
                          AppendParams& p) {
  if (!k_new || !v_new) return fail(NIYAMA_EINVAL, "k_new/v_new is NULL");
  if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15)
    return fail(NIYAMA_EINVAL, "k_new/v_new must be 16-byte aligned");
  p = AppendParams{};
  p.pool_k = kv->pool + static_cast<int64_t>(layer) * 2 * kv->half_bytes;
  p.pool_v = p.pool_k + kv->v_offset;
  p.k_new = static_cast<const uint8_t*>(k_new);
  p.v_new = static_cast<const uint8_t*>(v_new);
  p.slot_map = plan->d_slot;
  p.chunk_bytes = kv->chunk_bytes;
  p.chunk_stride = kv->chunk_stride;
  p.T = plan->T;
  p.Hkv = kv->hkv;
  p.row_bytes = kv->row_bytes;
  p.B = kv->B;
  p.v_t = kv->cfg.dtype == NIYAMA_BF16 ? 1 : 0;
  p.vgrp = plan->d_vgrp;
  p.velem = plan->d_velem;
  p.n_grp = static_cast<int32_t>(plan->vgrp.size());
  p.n_elem = static_cast<int32_t>(plan->velem.size());
  // the plan's freshly uploaded metadata (block tables, unit queue, ...) into L2 while the
  // append runs, so the attention launch that follows does not start on cold plan data
  p.pf_base = plan->dbuf;
  p.pf_bytes = static_cast<uint32_t>(std::min<size_t>(plan->meta_bytes, size_t(64) << 20) & ~size_t(15));
  return NIYAMA_OK;
}

int64_t append_pieces(const AppendParams& p) {
  const int64_t pieces = p.row_bytes >> 4;
  return static_cast<int64_t>(p.T) * p.Hkv * pieces +
         (p.v_t ? static_cast<int64_t>(p.n_grp) * p.Hkv * (p.row_bytes >> 1) + static_cast<int64_t>(p.n_elem) * p.Hkv * pieces
                : 0);
}

niyama_status attention_impl(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* q, void* o, float* lse,
                             float softmax_scale, niyama_stream stream, const AppendParams* ap,
                             const AttnParams::Gather* gx = nullptr);
}  // namespace

extern "C" niyama_status niyama_kv_append(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* k_new,
                                          const void* v_new, niyama_stream stream) {
  niyama_status st = check_launch(kv, plan, layer);
  if (st != NIYAMA_OK) return st;
  if (plan->T == 0) return NIYAMA_OK;
  AppendParams p{};
  st = fill_append(kv, plan, layer, k_new, v_new, p);
  if (st != NIYAMA_OK) return st;
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  NY_CUDA(wait_plan(plan, stream));
  NY_CUDA(launch_append(p, reinterpret_cast<cudaStream_t>(stream)));
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_append_attention(niyama_kv* kv, const niyama_plan* plan, int32_t layer,
                                                 const void* k_new, const void* v_new, const void* q, void* o,
                                                 float* lse, float softmax_scale, niyama_stream stream) {
  niyama_status st = check_launch(kv, plan, layer);
  if (st != NIYAMA_OK) return st;
  if (plan->T == 0) return NIYAMA_OK;
  if (kv->cfg.dtype != NIYAMA_BF16) {  // f32 (config 1): the two launches
    st = niyama_kv_append(kv, plan, layer, k_new, v_new, stream);
    return st != NIYAMA_OK ? st : niyama_hybrid_attention(kv, plan, layer, q, o, lse, softmax_scale, stream);
  }
  AppendParams ap{};
  st = fill_append(kv, plan, layer, k_new, v_new, ap);
  if (st != NIYAMA_OK) return st;
  if (append_pieces(ap) >= (int64_t(1) << 31)) return fail(NIYAMA_EINVAL, "append: too many pieces");
  return attention_impl(kv, plan, layer, q, o, lse, softmax_scale, stream, &ap);
}

extern "C" niyama_status niyama_hybrid_attention(niyama_kv* kv, const niyama_plan* plan, int32_t layer,
                                                 const void* q, void* o, float* lse, float softmax_scale,
                                                 niyama_stream stream) {
  niyama_status st = check_launch(kv, plan, layer);
  if (st != NIYAMA_OK) return st;
  if (plan->T == 0) return NIYAMA_OK;
  return attention_impl(kv, plan, layer, q, o, lse, softmax_scale, stream, nullptr);
}

namespace {
niyama_status attention_impl(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* q, void* o, float* lse,
                             float softmax_scale, niyama_stream stream, const AppendParams* ap,
                             const AttnParams::Gather* gx) {
  if (!q || !o) return fail(NIYAMA_EINVAL, "q/o is NULL");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(o)) & 15)
    return fail(NIYAMA_EINVAL, "q/o must be 16-byte aligned");
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(static_cast<float>(kv->d));
  AttnParams p{};
  p.pool_k = kv->pool + static_cast<int64_t>(layer) * 2 * kv->half_bytes;
  p.pool_v = p.pool_k + kv->v_offset;
  p.q = q;
  p.o = o;
  p.lse = lse;
  p.tables = plan->d_tables;
  p.slices = plan->d_slices;
  p.drows = plan->d_drows;
  p.rows = plan->d_rows;
  p.part_o = plan->d_part_o;
  p.part_ml = plan->d_part_ml;
  p.ppart_o = plan->d_ppart_o;
  p.ppart_ml = plan->d_ppart_ml;
  p.pcounters = plan->d_pcounters;
  p.work = plan->d_work;
  p.chunk_bytes = kv->chunk_bytes;
  p.chunk_stride = kv->chunk_stride;
  p.kv_adjacent = kv->v_offset == kv->chunk_bytes ? 1 : 0;
  // g <= 4: 12 decode warps x 2-stage rings; g = 8 (twice the MMA work per byte): 8 x 3
  // (measured: config 2 102.6 -> 99.4 us with 12; config 4 1180 -> 1218 us with 12)
  p.dec_warps = decode_streams(kv->g, kv->tune.decode_path);
  // decode_path 0 = auto: producer warps at g = 8 (the 4 warps a 3-stage ring layout leaves
  // idle; config 4 870 -> 850 us), per-warp loaders at g <= 4 (12 compute warps measured
  // faster: config 2 96.3 vs 98.4 us with 8 + 4); kernel modes 0 per-warp, 1 tcgen05, 2 producer
  {
    const int dp = kv->tune.decode_path;
    p.dec_mode = dp == 1 ? 1 : (dp == 2 || (dp == 0 && kv->g > 4)) ? 2 : 0;
  }
  p.T = plan->T;
  p.Hq = kv->hq;
  p.Hkv = kv->hkv;
  p.d = kv->d;
  p.B = kv->B;
  p.g = kv->g;
  p.b_shift = __builtin_ctz(static_cast<unsigned>(kv->B));
  p.hkv_shift = (kv->hkv & (kv->hkv - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(kv->hkv)) : -1;
  p.R = plan->R;
  p.n_tiles = plan->n_tiles;
  p.n_units = plan->n_units;
  p.n_slices = static_cast<int32_t>(plan->slices.size());
  p.n_drows = static_cast<int32_t>(plan->drows.size());
  p.split_len = plan->split_len;
  p.uq = plan->d_uq;
  p.mq = plan->d_mq;
  p.counters = plan->d_counters;
  p.epoch = plan->launches;
  p.n_merge_rows = plan->n_merge_rows;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = kv->trace;
  if (ap) {
    p.ap = *ap;
    p.append_total = static_cast<int32_t>(append_pieces(*ap));
  }
  if (gx) p.gx = *gx;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  NY_CUDA(wait_plan(plan, stream));
  if (kv->cfg.dtype == NIYAMA_BF16) {  // shapes checked at niyama_kv_create
    int grid = kv->tune.grid_cap > 0 ? std::min(kv->tune.grid_cap, plan->grid) : plan->grid;
    p.prefill_ctas = std::min(plan->prefill_ctas, grid);
    const bool pairs = kv->tune.prefill_pairs == 1 || (kv->tune.prefill_pairs == 0 && kv->g > 4);
    // an odd grid grows by one CTA (never past the SM count or a grid_cap) or shrinks by one:
    // the queues hand work to whichever CTAs run, so the CTA count changes no result
    const int cap = kv->tune.grid_cap > 0 ? std::min(kv->tune.grid_cap, kv->num_sms) : kv->num_sms;
    const int even_grid = (grid & 1) && grid + 1 <= cap ? grid + 1 : grid & ~1;
    if (pairs && plan->n_tiles > 0 && plan->n_split_tiles == 0 && even_grid >= 2) {
      // CTA pairs: clusters of 2 (even grid, even prefill CTA count), one item per q-tile pair
      // (auto at g = 8: config 4 866 -> 849 us; neutral at g = 4, tools/ab_pairs.py)
      p.pairs = 1;
      p.n_pair_items = 0;
      for (const PrefillSlice& sl : plan->slices) p.n_pair_items += (sl.nqt + 1) / 2 * kv->hkv;
      grid = even_grid;
      p.prefill_ctas = std::min(grid, std::max(2, p.prefill_ctas + (p.prefill_ctas & 1)));
    }
    NY_CUDA(launch_attention_bf16(p, grid, s));
    ++plan->launches;
  } else {
    NY_CUDA(launch_attention_generic_f32(p, s));
  }
  return NIYAMA_OK;
}
}  // namespace

extern "C" niyama_status niyama_debug_trace(niyama_kv* kv, int64_t* device_buf) {
  if (!kv) return fail(NIYAMA_EINVAL, "kv is NULL");
  kv->trace = device_buf;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_get_tuning(const niyama_kv* kv, niyama_tuning* out) {
  if (!kv || !out) return fail(NIYAMA_EINVAL, "kv/out is NULL");
  *out = kv->tune;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_kv_set_tuning(niyama_kv* kv, const niyama_tuning* t) {
  if (!kv || !t) return fail(NIYAMA_EINVAL, "kv/tuning is NULL");
  if (t->prefill_ctas < 0 || t->grid_cap < 0) return fail(NIYAMA_EINVAL, "tuning: prefill_ctas/grid_cap < 0");
  if (t->decode_path < 0 || t->decode_path > 3) return fail(NIYAMA_EINVAL, "tuning: decode_path must be 0-3");
  if (t->prefill_split != 0 && t->prefill_split != 1) return fail(NIYAMA_EINVAL, "tuning: prefill_split must be 0 or 1");
  if (t->prefill_pairs < 0 || t->prefill_pairs > 2) return fail(NIYAMA_EINVAL, "tuning: prefill_pairs must be 0-2");
  if (t->split_len != 0 && (t->split_len < 16 || t->split_len % 16)) return fail(NIYAMA_EINVAL, "tuning: split_len");
  if (t->tail_div < 1 || t->tail_div > 16) return fail(NIYAMA_EINVAL, "tuning: tail_div outside [1, 16]");
  if (t->tail_min < 16 || t->tail_min % 16) return fail(NIYAMA_EINVAL, "tuning: tail_min must be a multiple of 16");
  if (t->plan_copy_stream != 0 && t->plan_copy_stream != 1) return fail(NIYAMA_EINVAL, "tuning: plan_copy_stream");
  kv->tune = *t;
  return NIYAMA_OK;
}

// ================================================================ NCCL (a7)
extern "C" niyama_status niyama_get_unique_id(void* out128) {
  if (!out128) return fail(NIYAMA_EINVAL, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NY_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_comm_init(niyama_kv* kv, const void* nccl_unique_id) {
  if (!kv || !nccl_unique_id) return fail(NIYAMA_EINVAL, "kv/unique_id is NULL");
  if (!kv->has_device) return fail(NIYAMA_EUNSUPPORTED, "no device");
  if (kv->comm) return fail(NIYAMA_EINVAL, "communicator already initialised");
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  NY_NCCL(ncclCommInitRank(&kv->comm, kv->cfg.world_size, id, kv->cfg.rank));
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_allgather_heads(niyama_kv* kv, const niyama_plan* plan, void* o_full,
                                                float* lse_full, niyama_stream stream) {
  niyama_status st = check_launch(kv, plan, 0);
  if (st != NIYAMA_OK) return st;
  if (!o_full) return fail(NIYAMA_EINVAL, "o_full is NULL");
  if (!kv->comm) return fail(NIYAMA_EINVAL, "niyama_comm_init was not called");
  if (plan->T == 0) return NIYAMA_OK;
  // The collective runs at every world size (at 1 it is NCCL's in-place copy), so the
  // single-GPU path exercises the same call a sharded job makes.
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  const size_t count = static_cast<size_t>(kv->hq) * plan->T * kv->d;
  uint8_t* base = static_cast<uint8_t*>(o_full);
  const ncclDataType_t ty = kv->cfg.dtype == NIYAMA_BF16 ? ncclBfloat16 : ncclFloat32;
  // Every grouped call is issued and the group always closed, even after an error (an
  // open group would capture the thread's later NCCL calls, torch's included).
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return fail(NIYAMA_ENCCL, std::string("ncclGroupStart: ") + ncclGetErrorString(r));
  ncclResult_t first = ncclAllGather(base + count * kv->elt * kv->cfg.rank, base, count, ty, kv->comm, s);
  if (lse_full) {
    const size_t lc = static_cast<size_t>(kv->hq) * plan->T;
    const ncclResult_t r2 = ncclAllGather(lse_full + lc * kv->cfg.rank, lse_full, lc, ncclFloat32, kv->comm, s);
    if (first == ncclSuccess) first = r2;
  }
  r = ncclGroupEnd();
  if (first == ncclSuccess) first = r;
  if (first != ncclSuccess) return fail(NIYAMA_ENCCL, std::string("all-gather: ") + ncclGetErrorString(first));
  return NIYAMA_OK;
}

// ================================================ §8(f)2 fused all-gather window
// One NCCL symmetric window per gather object: [buffer 0 | buffer 1 | flags], each buffer
// o_full [Hq_all][max_rows][d] bf16 then lse_full [Hq_all][max_rows] f32, 4 KB aligned.
struct niyama_gather {
  niyama_kv* kv = nullptr;
  uint8_t* base = nullptr;
  size_t bytes = 0, o_bytes = 0, buf_bytes = 0, flags_off = 0;
  ncclWindow_t win = nullptr;
  int32_t max_rows = 0;
  uint32_t epoch = 0;
  bool nccl_owned = true;  // false: niyama_debug_gather_group (cudaMalloc, one process)
  AttnParams::Gather gx{};
};

namespace {
size_t align4k(size_t x) { return (x + 4095) & ~static_cast<size_t>(4095); }

void gather_release(niyama_gather* g) {
  if (g->win) ncclCommWindowDeregister(g->kv->comm, g->win);
  if (g->base) {
    if (g->nccl_owned)
      ncclMemFree(g->base);
    else
      cudaFree(g->base);
  }
  delete g;
}

niyama_gather* gather_layout(niyama_kv* kv, int32_t max_rows) {
  auto* g = new niyama_gather;
  g->kv = kv;
  g->max_rows = max_rows;
  const size_t rows_all = static_cast<size_t>(kv->hq) * kv->cfg.world_size * max_rows;
  g->o_bytes = align4k(rows_all * kv->d * 2);
  g->buf_bytes = g->o_bytes + align4k(rows_all * sizeof(float));
  g->flags_off = 2 * g->buf_bytes;
  g->bytes = g->flags_off + 4096;
  return g;
}

niyama_status gather_check(niyama_kv* kv, int32_t max_rows) {
  if (!kv->has_device) return fail(NIYAMA_EUNSUPPORTED, "no device");
  if (kv->cfg.dtype != NIYAMA_BF16) return fail(NIYAMA_EINVAL, "the fused all-gather needs a bf16 pool");
  if (max_rows <= 0) return fail(NIYAMA_EINVAL, "max_rows must be > 0");
  if (kv->cfg.world_size > kMaxGatherRanks) return fail(NIYAMA_EUNSUPPORTED, "more ranks than one NVLink node (8)");
  return NIYAMA_OK;
}
}  // namespace

extern "C" niyama_status niyama_gather_create(niyama_kv* kv, int32_t max_rows, niyama_gather** out) {
  if (!kv || !out) return fail(NIYAMA_EINVAL, "kv/out is NULL");
  *out = nullptr;
  niyama_status st = gather_check(kv, max_rows);
  if (st != NIYAMA_OK) return st;
  if (!kv->comm) return fail(NIYAMA_EINVAL, "niyama_comm_init was not called");
  const int world = kv->cfg.world_size;
  DeviceGuard dg(kv->cfg.device);
  NY_CUDA(dg.err);
  niyama_gather* g = gather_layout(kv, max_rows);
  void* base = nullptr;
  ncclResult_t r = ncclMemAlloc(&base, g->bytes);
  if (r != ncclSuccess) {
    delete g;
    return fail(NIYAMA_EUNSUPPORTED, std::string("ncclMemAlloc: ") + ncclGetErrorString(r));
  }
  g->base = static_cast<uint8_t*>(base);
  // zeroed (flags at epoch 0) and complete before this rank joins the collective
  // registration, so no peer's first launch can meet an uninitialised flag
  cudaError_t ce = cudaMemset(g->base, 0, g->bytes);
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    gather_release(g);
    return fail(NIYAMA_ECUDA, std::string("window init: ") + cudaGetErrorString(ce));
  }
  r = ncclCommWindowRegister(kv->comm, g->base, g->bytes, &g->win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess || !g->win) {
    g->win = nullptr;
    gather_release(g);
    return fail(NIYAMA_EUNSUPPORTED, std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r));
  }
  uint64_t peers[kMaxGatherRanks] = {};
  ce = gather_resolve_peers(g->win, world, peers);
  if (ce != cudaSuccess) {
    gather_release(g);
    return fail(NIYAMA_ECUDA, std::string("window peer mapping: ") + cudaGetErrorString(ce));
  }
  for (int i = 0; i < world; ++i) {
    if (peers[i] == 0) {
      gather_release(g);
      return fail(NIYAMA_EUNSUPPORTED, "the window has no load/store mapping of rank " + std::to_string(i));
    }
    g->gx.delta[i] = static_cast<int64_t>(peers[i] - reinterpret_cast<uint64_t>(g->base));
  }
  g->gx.n = world;
  g->gx.rank = kv->cfg.rank;
  g->gx.flags = reinterpret_cast<uint32_t*>(g->base + g->flags_off);
  *out = g;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_debug_gather_group(niyama_kv* const* kvs, int32_t n, int32_t max_rows,
                                                   niyama_gather** outs) {
  if (!kvs || !outs || n < 1 || n > kMaxGatherRanks) return fail(NIYAMA_EINVAL, "kvs/outs NULL or n out of [1, 8]");
  for (int32_t r = 0; r < n; ++r) {
    outs[r] = nullptr;
    if (!kvs[r]) return fail(NIYAMA_EINVAL, "kvs[r] is NULL");
    niyama_status st = gather_check(kvs[r], max_rows);
    if (st != NIYAMA_OK) return st;
    if (kvs[r]->cfg.world_size != n || kvs[r]->cfg.rank != r || kvs[r]->cfg.device != kvs[0]->cfg.device ||
        kvs[r]->hq != kvs[0]->hq || kvs[r]->d != kvs[0]->d)
      return fail(NIYAMA_EINVAL, "kvs[r] must be rank r of world n, one device, one shape");
  }
  DeviceGuard dg(kvs[0]->cfg.device);
  NY_CUDA(dg.err);
  niyama_gather* gs[kMaxGatherRanks] = {};
  cudaError_t ce = cudaSuccess;
  for (int32_t r = 0; r < n && ce == cudaSuccess; ++r) {
    gs[r] = gather_layout(kvs[r], max_rows);
    gs[r]->nccl_owned = false;
    void* base = nullptr;
    ce = cudaMalloc(&base, gs[r]->bytes);
    gs[r]->base = static_cast<uint8_t*>(base);
    if (ce == cudaSuccess) ce = cudaMemset(base, 0, gs[r]->bytes);
  }
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    for (int32_t r = 0; r < n; ++r)
      if (gs[r]) gather_release(gs[r]);
    return fail(NIYAMA_ECUDA, std::string("debug gather group: ") + cudaGetErrorString(ce));
  }
  for (int32_t r = 0; r < n; ++r) {
    for (int32_t i = 0; i < n; ++i)
      gs[r]->gx.delta[i] = reinterpret_cast<intptr_t>(gs[i]->base) - reinterpret_cast<intptr_t>(gs[r]->base);
    gs[r]->gx.n = n;
    gs[r]->gx.rank = r;
    gs[r]->gx.flags = reinterpret_cast<uint32_t*>(gs[r]->base + gs[r]->flags_off);
    outs[r] = gs[r];
  }
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_gather_destroy(niyama_gather* g) {
  if (!g) return NIYAMA_OK;
  DeviceGuard dg(g->kv->cfg.device);
  NY_CUDA(dg.err);
  const cudaError_t ce = cudaDeviceSynchronize();
  gather_release(g);
  if (ce != cudaSuccess) return fail(NIYAMA_ECUDA, std::string("gather destroy: ") + cudaGetErrorString(ce));
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_attention_gather(niyama_kv* kv, const niyama_plan* plan, int32_t layer,
                                                 const void* k_new, const void* v_new, const void* q,
                                                 niyama_gather* g, float softmax_scale, void** o_full,
                                                 float** lse_full, niyama_stream stream) {
  niyama_status st = check_launch(kv, plan, layer);
  if (st != NIYAMA_OK) return st;
  if (!g || !o_full || !lse_full) return fail(NIYAMA_EINVAL, "gather/o_full/lse_full is NULL");
  if (g->kv != kv) return fail(NIYAMA_EINVAL, "the gather window belongs to another niyama_kv");
  if (plan->T > g->max_rows) return fail(NIYAMA_EINVAL, "plan rows exceed the window's max_rows");
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(NIYAMA_EINVAL, "k_new and v_new: both or neither");
  AppendParams ap{};
  if (k_new) {
    st = fill_append(kv, plan, layer, k_new, v_new, ap);
    if (st != NIYAMA_OK) return st;
    if (append_pieces(ap) >= (int64_t(1) << 31)) return fail(NIYAMA_EINVAL, "append: too many pieces");
  }
  const uint32_t epoch = g->epoch + 1;
  uint8_t* buf = g->base + (epoch & 1) * g->buf_bytes;
  const int64_t T = plan->T;
  uint8_t* o = buf + static_cast<int64_t>(kv->cfg.rank) * kv->hq * T * kv->d * 2;
  float* lse = reinterpret_cast<float*>(buf + g->o_bytes) + static_cast<int64_t>(kv->cfg.rank) * kv->hq * T;
  if (T > 0) {
    AttnParams::Gather gx = g->gx;
    gx.epoch = epoch;
    st = attention_impl(kv, plan, layer, q, o, lse, softmax_scale, stream, k_new ? &ap : nullptr, &gx);
    if (st != NIYAMA_OK) return st;
    g->epoch = epoch;
  }
  *o_full = buf;
  *lse_full = reinterpret_cast<float*>(buf + g->o_bytes);
  return NIYAMA_OK;
}

// ================================================================ slack (a1)
extern "C" niyama_status niyama_min_slack(const niyama_decode_qos* decodes, int32_t n, double now, double* slack_out) {
  if (!slack_out || n < 0 || (n > 0 && !decodes)) return fail(NIYAMA_EINVAL, "NULL argument or n < 0");
  double s = std::numeric_limits<double>::infinity();
  for (int32_t i = 0; i < n; ++i) {
    const niyama_decode_qos& q = decodes[i];
    double si;
    if (q.interactive) {
      if (q.next_token < 1) return fail(NIYAMA_EINVAL, "next_token < 1 (Eq. 2 needs n >= 1)");
      si = q.t_arrival + q.slo_ttft + (q.next_token - 1) * q.slo_tbt - now;  // Eq. 2
    } else {
      si = (q.t_arrival + q.slo_ttlt - now) / std::max(1, q.est_remaining);  // Eq. 3, pacing bound
    }
    s = std::min(s, si);
  }
  *slack_out = s;
  return NIYAMA_OK;
}
