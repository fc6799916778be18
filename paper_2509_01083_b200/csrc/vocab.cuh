// vocab.cuh — vocabulary-parallel (tensor-parallel LM head) verification,
// SURVEY §8(f) f3 (a 70B target on 8 GPUs implies a
// vocab-parallel LM head). Included by verify.cu inside its translation unit
// (after the kernels it reuses).
//
// Shard s of n holds the columns [v0_s, v0_s + Vs_s) of every target and
// draft row, v0_s = s W with W a multiple of the 2048-token stream slice (512
// for fp32) and the last shard taking the remainder. The stages, with the
// caller's collectives in between (dsde_vp_verify runs them over NCCL):
//   1. dsde_vp_stream   (per shard) the stream slices of its columns -> its
//                       block of the partials [n][total][ns_sh]; the owner of
//                       each draft token x writes (t_x, d_x), the others 0;
//      -> all-gather the partial blocks, all-reduce (sum) the (t_x, d_x)
//   2. dsde_vp_finalize (every shard, identically) the fp64 row merge over
//                       all slices, KL, accept test, first rejection, layout
//                       and the draw record of every sequence;
//   3. dsde_vp_draw     (per shard) the draw masses of its draw slices of each
//                       sequence's drawn row -> its block [n][B][nd_sh];
//      -> all-gather the mass blocks
//   4. dsde_vp_select   (every shard) R and the crossing slice over all
//                       masses; the owner of that slice scans it -> the
//                       token (global id, flags << 24), the others -1;
//      -> all-reduce (max) the tokens
//   5. dsde_vp_place    (every shard) the drawn tokens into emitted / flags.
// The shard boundaries are slice boundaries, so every partial and mass is
// bit-identical to the unsharded pass's, and stages 2 and 4 read them in the
// unsharded order: the outputs are bit-identical to dsde_verify's.
// Supported: sampling at T = 1 with the D7 recovery draw (dsde_config.resample
// = DSDE_RESAMPLE_FULL; no greedy, no temperature, no masks, no draft entropy,
// no device_rows): DSDE_ERR_ARG otherwise.

namespace dsde {

struct VpMass {  // one draw slice's record in the exchange buffer (16 bytes)
  double m;
  float ref;
  int pad;
};
static_assert(sizeof(VpMass) == 16, "VpMass layout");

template <typename T>
constexpr int vp_align() {  // shard width granularity: one stream slice
  return sub_elems<T>();
}

inline int vp_width(int V, int nshards, dsde_dtype dt) {
  const int g = dt == DSDE_BF16 ? vp_align<uint16_t>() : vp_align<float>();
  const int w = (V + nshards - 1) / nshards;
  return (w + g - 1) / g * g;
}

// (t_x, d_x) of every draft row whose token this shard owns, (0, 0) elsewhere.
template <typename T>
__global__ void k_vp_xlog(int B, int total, const int32_t* cu_sl, const int32_t* tokens, const T* tl,
                          long long ld_t, const T* dl, long long ld_d, int v0, int Vs, float2* xlog) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= total) return;
  // the row's sequence: the last i with cu_sl[i] <= r
  int lo = 0, hi = B - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(cu_sl + mid) <= r) lo = mid;
    else hi = mid - 1;
  }
  const int x = __ldg(tokens + r) - v0;
  float2 g = make_float2(0.f, 0.f);
  if (x >= 0 && x < Vs) g = make_float2(load_logit<T>(tl + (long long)(r + lo) * ld_t + x),
                                        load_logit<T>(dl + (long long)r * ld_d + x));
  xlog[r] = g;
}

// Draw masses of this shard's draw slices: one warp per (sequence, slice).
template <typename T>
__global__ void __launch_bounds__(256) k_vp_draw(int B, int Vs, int nd_sh, const SeqRec* rec, const T* tl,
                                                 long long ld_t, const T* dl, long long ld_d, VpMass* out) {
  const long long W = (long long)gridDim.x * 8;
  for (long long q = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); q < (long long)B * nd_sh; q += W) {
    const int i = (int)(q / nd_sh), u = (int)(q - (long long)i * nd_sh);
    const SeqRec r = load_seqrec(rec + i);
    VpMass* o = out + q;
    if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) {
      if ((threadIdx.x & 31) == 0) *o = VpMass{0.0, -INFINITY, 0};
      continue;
    }
    double m;
    float ref;
    draw_mass<T>(r, u, Vs, tl, ld_t, dl, ld_d, &m, &ref);
    if ((threadIdx.x & 31) == 0) *o = VpMass{m, ref, 0};
  }
}

// Slice records of the gathered mass blocks [n][B][nd_sh] (global slice s).
struct VpSrc {
  const VpMass* all;
  int i, B, nd_sh;
  __device__ __forceinline__ const VpMass* at(int s) const {
    const int b = s / nd_sh;
    return all + ((long long)b * B + i) * nd_sh + (s - b * nd_sh);
  }
  __device__ __forceinline__ double m(int s) const { return __ldcg(&at(s)->m); }
  __device__ __forceinline__ float r(int s) const { return __ldcg(&at(s)->ref); }
  const double* scale = nullptr;
};

// select_seq over the gathered masses (its SliceSrc<false> accessors, sharded).
template <typename T>
__global__ void __launch_bounds__(128) k_vp_select(SelArgs a, const SeqRec* rec, const VpMass* all) {
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= a.B) return;
  const SeqRec r = load_seqrec(rec + i);
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) {
    if ((threadIdx.x & 31) == 0) a.tok_out[i] = -1;
    return;
  }
  select_seq<T, false, VpSrc>(a, i, r, VpSrc{all, i, a.B, a.nd_sh});
}

// The drawn tokens (all-reduced) into emitted / flags.
__global__ void k_vp_place(int B, const SeqRec* rec, const int32_t* tok, int32_t* emitted, uint8_t* flags,
                           int32_t* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const SeqRec r = rec[i];
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) return;
  const int v = tok[i];
  if (v < 0) {  // no shard selected (a stage failed): reported by the select
    emitted[r.slot] = DSDE_PAD;
    return;
  }
  emitted[r.slot] = v & 0xffffff;
  if (flags) flags[r.slot] |= (uint8_t)((unsigned)v >> 24);
}

}  // namespace dsde

extern "C" dsde_status dsde_vp_sizes(int V, int nshards, dsde_dtype dtype, int* shard_width, int* ns_sh,
                                     int* nd_sh) {
  if (V < 2 || nshards < 1 || (dtype != DSDE_F32 && dtype != DSDE_BF16) || !shard_width || !ns_sh || !nd_sh)
    return DSDE_ERR_ARG;
  const int W = vp_width(V, nshards, dtype);
  if ((long long)W * (nshards - 1) >= V) return DSDE_ERR_ARG;  // every shard non-empty
  *shard_width = W;
  *ns_sh = W / (dtype == DSDE_BF16 ? sub_elems<uint16_t>() : sub_elems<float>());
  *nd_sh = W / (dtype == DSDE_BF16 ? draw_elems<uint16_t>() : draw_elems<float>());
  return DSDE_OK;
}

namespace {
struct VpShape {
  int W, ns_sh, nd_sh, v0, Vs;
};
dsde_status vp_shape(int V, int nshards, int shard, dsde_dtype dt, VpShape* o) {
  if (shard < 0 || shard >= nshards) return DSDE_ERR_ARG;
  const dsde_status s = dsde_vp_sizes(V, nshards, dt, &o->W, &o->ns_sh, &o->nd_sh);
  if (s != DSDE_OK) return s;
  o->v0 = shard * o->W;
  o->Vs = std::min(o->W, V - o->v0);
  return DSDE_OK;
}
bool vp_mode_ok(dsde_state st) {
  return st && !st->cfg.greedy && !st->cfg.masked && !st->cfg.device_rows && !st->temps && !st->entropy_out &&
         st->cfg.resample == DSDE_RESAMPLE_FULL;
}
}  // namespace

extern "C" dsde_status dsde_vp_stream(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype,
                                      int total_draft_rows, const int32_t* cu_sl, const int32_t* draft_tokens,
                                      const void* target_shard, int64_t ld_t, const void* draft_shard,
                                      int64_t ld_d, void* part_block, float* xlog, void* stream) {
  VpShape sh;
  if (!vp_mode_ok(st) || !cu_sl || !draft_tokens || !target_shard || !draft_shard || !part_block || !xlog)
    return DSDE_ERR_ARG;
  if (vp_shape(V, nshards, shard, dtype, &sh) != DSDE_OK) return DSDE_ERR_ARG;
  if (B < 1 || total_draft_rows < B || total_draft_rows > B * DSDE_MAX_SL || ld_t < sh.Vs || ld_d < sh.Vs)
    return DSDE_ERR_ARG;
  const size_t esz = dtype == DSDE_BF16 ? 2 : 4;
  if ((((uintptr_t)target_shard) | ((uintptr_t)draft_shard) | ((uintptr_t)part_block)) & 15) return DSDE_ERR_ARG;
  if (((size_t)ld_t * esz) % 16 || ((size_t)ld_d * esz) % 16) return DSDE_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StreamArgs sa{target_shard, ld_t, draft_shard, ld_d, cu_sl, B, sh.Vs, sh.ns_sh, total_draft_rows,
                reinterpret_cast<SubPartial*>(part_block), 0, nullptr, nullptr};
  const int sms = sm_count();
  const int nthr = 256, nb = (total_draft_rows + nthr - 1) / nthr;
  if (dtype == DSDE_BF16) {
    static int g = 0;
    if (!g) g = sms * resident_per_sm(k_stream_ldg<uint16_t, false, false>, kLdgThreads);
    k_stream_ldg<uint16_t, false, false><<<g, kLdgThreads, 0, s>>>(sa);
    k_vp_xlog<uint16_t><<<nb, nthr, 0, s>>>(B, total_draft_rows, cu_sl, draft_tokens,
                                            reinterpret_cast<const uint16_t*>(target_shard), ld_t,
                                            reinterpret_cast<const uint16_t*>(draft_shard), ld_d, sh.v0, sh.Vs,
                                            reinterpret_cast<float2*>(xlog));
  } else {
    static int g = 0;
    if (!g) g = sms * resident_per_sm(k_stream_ldg<float, false, false>, kLdgThreads);
    k_stream_ldg<float, false, false><<<g, kLdgThreads, 0, s>>>(sa);
    k_vp_xlog<float><<<nb, nthr, 0, s>>>(B, total_draft_rows, cu_sl, draft_tokens,
                                         reinterpret_cast<const float*>(target_shard), ld_t,
                                         reinterpret_cast<const float*>(draft_shard), ld_d, sh.v0, sh.Vs,
                                         reinterpret_cast<float2*>(xlog));
  }
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_vp_finalize(dsde_state st, int B, int V, int nshards, dsde_dtype dtype,
                                        int total_draft_rows, const int32_t* cu_sl, const int32_t* draft_tokens,
                                        const void* part_all, const float* xlog, const uint64_t* seeds,
                                        int32_t* accepted_len, int32_t* emitted_tokens, float* kld,
                                        uint8_t* flags, void* rec, void* stream) {
  VpShape sh;
  if (!vp_mode_ok(st) || !cu_sl || !draft_tokens || !part_all || !xlog || !seeds || !accepted_len ||
      !emitted_tokens || !kld || !rec)
    return DSDE_ERR_ARG;
  if (vp_shape(V, nshards, 0, dtype, &sh) != DSDE_OK) return DSDE_ERR_ARG;
  if (B < 1 || total_draft_rows < B || total_draft_rows > B * DSDE_MAX_SL) return DSDE_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TailArgs p{};
  const int ns = n_subs(V, dtype);
  // tl / dl are not read (t_x, d_x come from xlog; no draw here)
  p.fa = FinArgs{B, V, total_draft_rows, ns, cu_sl, draft_tokens, nullptr, 0, nullptr, 0, seeds,
                 reinterpret_cast<const SubPartial*>(part_all), accepted_len, emitted_tokens, kld, flags,
                 reinterpret_cast<SeqRec*>(rec), st->err, 0, 0, nullptr, 0, nullptr, 0, sh.ns_sh,
                 (long long)total_draft_rows * sh.ns_sh, reinterpret_cast<const float2*>(xlog)};
  p.no_draw = 1;
  if (dtype == DSDE_BF16) launch_tail<uint16_t>(p, B, s);
  else launch_tail<float>(p, B, s);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_vp_draw(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype,
                                    const void* rec, const void* target_shard, int64_t ld_t,
                                    const void* draft_shard, int64_t ld_d, void* mass_block, void* stream) {
  VpShape sh;
  if (!vp_mode_ok(st) || !rec || !target_shard || !draft_shard || !mass_block) return DSDE_ERR_ARG;
  if (vp_shape(V, nshards, shard, dtype, &sh) != DSDE_OK || B < 1) return DSDE_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = std::min((long long)sm_count() * 8, ((long long)B * sh.nd_sh + 7) / 8);
  if (dtype == DSDE_BF16)
    k_vp_draw<uint16_t><<<grid, 256, 0, s>>>(B, sh.Vs, sh.nd_sh, reinterpret_cast<const SeqRec*>(rec),
                                             reinterpret_cast<const uint16_t*>(target_shard), ld_t,
                                             reinterpret_cast<const uint16_t*>(draft_shard), ld_d,
                                             reinterpret_cast<VpMass*>(mass_block));
  else
    k_vp_draw<float><<<grid, 256, 0, s>>>(B, sh.Vs, sh.nd_sh, reinterpret_cast<const SeqRec*>(rec),
                                          reinterpret_cast<const float*>(target_shard), ld_t,
                                          reinterpret_cast<const float*>(draft_shard), ld_d,
                                          reinterpret_cast<VpMass*>(mass_block));
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_vp_select(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype,
                                      const void* rec, const void* mass_all, const void* target_shard,
                                      int64_t ld_t, const void* draft_shard, int64_t ld_d, int32_t* tok_out,
                                      void* stream) {
  VpShape sh;
  if (!vp_mode_ok(st) || !rec || !mass_all || !target_shard || !draft_shard || !tok_out) return DSDE_ERR_ARG;
  if (vp_shape(V, nshards, shard, dtype, &sh) != DSDE_OK || B < 1) return DSDE_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nd = n_draws(V, dtype);
  SelArgs a{B, V, nd, target_shard, ld_t, draft_shard, ld_d, nullptr, nullptr, st->err, sh.v0,
            shard * sh.nd_sh, sh.nd_sh, sh.Vs, tok_out};
  if (dtype == DSDE_BF16)
    k_vp_select<uint16_t><<<(B + 3) / 4, 128, 0, s>>>(a, reinterpret_cast<const SeqRec*>(rec),
                                                      reinterpret_cast<const VpMass*>(mass_all));
  else
    k_vp_select<float><<<(B + 3) / 4, 128, 0, s>>>(a, reinterpret_cast<const SeqRec*>(rec),
                                                   reinterpret_cast<const VpMass*>(mass_all));
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_vp_place(dsde_state st, int B, const void* rec, const int32_t* tok_all,
                                     int32_t* emitted_tokens, uint8_t* flags, void* stream) {
  if (!st || B < 1 || !rec || !tok_all || !emitted_tokens) return DSDE_ERR_ARG;
  k_vp_place<<<(B + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      B, reinterpret_cast<const SeqRec*>(rec), tok_all, emitted_tokens, flags, st->err);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

// ---- the whole vocab-parallel verification over an NCCL communicator ----
dsde_status dsde_comm_allgather_bytes(dsde_comm comm, void* recv, size_t bytes, cudaStream_t s);
dsde_status dsde_comm_allreduce_f32_sum(dsde_comm comm, float* buf, size_t n, cudaStream_t s);
dsde_status dsde_comm_allreduce_i32_max(dsde_comm comm, int32_t* buf, size_t n, cudaStream_t s);
int dsde_comm_rank(dsde_comm comm);
int dsde_comm_size(dsde_comm comm);

namespace {
struct VpWs {
  char* part;     // [n][total][ns_sh] SubPartial
  float* xlog;    // [total][2]
  char* rec;      // [B] SeqRec
  char* mass;     // [n][B][nd_sh] VpMass
  int32_t* tok;   // [B]
  size_t part_blk, mass_blk, bytes;
};
VpWs vp_ws(int B, int total, const VpShape& sh, int n, char* base) {
  VpWs w{};
  w.part_blk = (size_t)32 * total * sh.ns_sh;
  w.mass_blk = (size_t)16 * B * sh.nd_sh;
  size_t o = 0;
  w.part = base + o;
  o += align256(w.part_blk * n);
  w.xlog = reinterpret_cast<float*>(base + o);
  o += align256((size_t)8 * total);
  w.rec = base + o;
  o += align256((size_t)64 * B);
  w.mass = base + o;
  o += align256(w.mass_blk * n);
  w.tok = reinterpret_cast<int32_t*>(base + o);
  o += align256((size_t)4 * B);
  w.bytes = o;
  return w;
}
}  // namespace

extern "C" size_t dsde_vp_workspace_size(int B, int total_draft_rows, int V, int nshards, dsde_dtype dtype) {
  VpShape sh;
  if (B < 1 || total_draft_rows < 0 || vp_shape(V, nshards, 0, dtype, &sh) != DSDE_OK) return 0;
  return vp_ws(B, total_draft_rows, sh, nshards, nullptr).bytes;
}

extern "C" dsde_status dsde_vp_verify(dsde_state st, int B, int V, dsde_dtype dtype, int total_draft_rows,
                                      const int32_t* cu_sl, const int32_t* draft_tokens, const void* target_shard,
                                      int64_t ld_t, const void* draft_shard, int64_t ld_d, const uint64_t* seeds,
                                      int32_t* accepted_len, int32_t* emitted_tokens, float* kld, uint8_t* flags,
                                      void* workspace, size_t ws_bytes, dsde_comm comm, void* stream) {
  NvtxRange nv("dsde_vp_verify");
  const int n = dsde_comm_size(comm), rank = dsde_comm_rank(comm);
  VpShape sh;
  if (!workspace || ((uintptr_t)workspace & 255) || vp_shape(V, n, rank, dtype, &sh) != DSDE_OK)
    return DSDE_ERR_ARG;
  const VpWs w = vp_ws(B, total_draft_rows, sh, n, reinterpret_cast<char*>(workspace));
  if (ws_bytes < w.bytes) return DSDE_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dsde_status r;
  // 1. this shard's partial block and x-logits, then the exchange
  if ((r = dsde_vp_stream(st, B, V, n, rank, dtype, total_draft_rows, cu_sl, draft_tokens, target_shard, ld_t,
                          draft_shard, ld_d, w.part + w.part_blk * rank, w.xlog, stream)) != DSDE_OK)
    return r;
  if (n > 1) {
    if ((r = dsde_comm_allgather_bytes(comm, w.part, w.part_blk, s)) != DSDE_OK) return r;
    if ((r = dsde_comm_allreduce_f32_sum(comm, w.xlog, (size_t)2 * total_draft_rows, s)) != DSDE_OK) return r;
  }
  // 2. the merge, accept test and layout (identical on every shard)
  if ((r = dsde_vp_finalize(st, B, V, n, dtype, total_draft_rows, cu_sl, draft_tokens, w.part, w.xlog, seeds,
                            accepted_len, emitted_tokens, kld, flags, w.rec, stream)) != DSDE_OK)
    return r;
  // 3. this shard's draw masses, then the exchange
  if ((r = dsde_vp_draw(st, B, V, n, rank, dtype, w.rec, target_shard, ld_t, draft_shard, ld_d,
                        w.mass + w.mass_blk * rank, stream)) != DSDE_OK)
    return r;
  if (n > 1 && (r = dsde_comm_allgather_bytes(comm, w.mass, w.mass_blk, s)) != DSDE_OK) return r;
  // 4. the select (the crossing slice's owner scans it), then the exchange
  if ((r = dsde_vp_select(st, B, V, n, rank, dtype, w.rec, w.mass, target_shard, ld_t, draft_shard, ld_d, w.tok,
                          stream)) != DSDE_OK)
    return r;
  if (n > 1 && (r = dsde_comm_allreduce_i32_max(comm, w.tok, (size_t)B, s)) != DSDE_OK) return r;
  // 5. the drawn tokens into the layout
  return dsde_vp_place(st, B, w.rec, w.tok, emitted_tokens, flags, stream);
}
