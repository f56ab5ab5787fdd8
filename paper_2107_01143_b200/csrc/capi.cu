// capi.cu — the extern "C" boundary (include/gvo_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "gvo_kernels.h"
#include "gvo_bytecode.cuh"

using namespace gvo;

namespace gvo {
// k_setup with geometry disabled: coefficient tables only (custom groups)
__global__ void k_coefs_only(TplView T, const gvo_config* cfgs, int64_t n, int64_t* coefs) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  const gvo_config cfg = cfgs[c];
  const int tpl = cfg.template_id;
  const int A = T.n_acc[tpl];
  const int abase = T.acc_base[tpl];
  const int64_t* fbase = T.field_base + T.field_base_off[tpl];
  const int32_t bd[3] = {cfg.block[0], cfg.block[1], cfg.block[2]};
  int64_t* crow = coefs + c * (int64_t)T.max_acc * 8;
  for (int a = lane; a < A; a += 32) {
    const int ga = abase + a;
    AffineForm f;
    int flag = affine_extract(T.code + T.code_off[ga], T.code_len[ga], bd, fbase, &f);
    for (int k = 0; k < 7; ++k) crow[a * 8 + k] = flag == kAffine ? f.c[k] : 0;
    crow[a * 8 + 7] = flag;
  }
}

__global__ void k_eval_addresses(TplView T, int tpl, int access, int32_t bx, int32_t by, int32_t bz,
                                 const int64_t* coords, int64_t n, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ga = T.acc_base[tpl] + access;
  const int32_t bd[3] = {bx, by, bz};
  int64_t crd[6];
  for (int k = 0; k < 6; ++k) crd[k] = coords[i * 6 + k];
  out[i] = eval_point(T.code + T.code_off[ga], T.code_len[ga], crd, bd,
                      T.field_base + T.field_base_off[tpl]);
}
}  // namespace gvo

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  bool ensure(size_t n) {
    if (n <= cap) return true;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, n * sizeof(T) + 16) != cudaSuccess) return false;
    cap = n;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct gvo_ctx {
  int device = 0;
  int n_sm = 148;
  std::string err;
  cudaStream_t stream = nullptr;
  // templates
  int n_tpl = 0;
  int max_fields = 0;
  int max_acc = 1;
  std::vector<int32_t> h_nacc, h_nfields;
  DBuf<int32_t> t_nf, t_na, t_ab, t_fbo, t_af, t_ak, t_co, t_cl, t_fko, t_fkl;
  DBuf<int64_t> t_fb, t_am;
  DBuf<int32_t> t_fcls, t_tcls;  // translation classes (k_dedup.cu)
  DBuf<gvo_insn> t_code;
  TplView view{};
  // machines
  std::vector<gvo_machine> h_machines;
  DBuf<gvo_machine> d_machines;
  DBuf<int32_t> d_mclass;  // machines with equal integer parameters share a class
  // cross-configuration sharing of identical set problems (k_dedup.cu):
  // GVO_DEDUP=0 evaluates every unit of every configuration
  bool dedup = true;
  // plan sharing across configurations (k_setup.cu): key table, leader
  // plan cache and per-batch sources, one table per call
  bool plan_share = true;
  DBuf<PlanEntry> plan_table;
  DBuf<int64_t> plan_cache, plan_src;
  DBuf<unsigned long long> plan_used;
  DBuf<uint8_t> plan_need;
  // gvo_sweep_host_ex with pinned host outputs: each batch's finished rows
  // are copied to the host on a second stream while later batches compute
  struct PipeOut {
    bool on = false;
    int64_t* counts = nullptr;
    double* stats = nullptr;
    double* records = nullptr;
    double* fd = nullptr;
    int64_t* l1 = nullptr;
    int32_t l1_stride = 0;
  } pipe;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  // work lists of the set kernel (k_dedup.cu k_worklist), per batch
  bool worklist = true;
  int64_t handoff_min = 1024;  // batches from this size hand large block units to the CTA (GVO_HANDOFF_MIN)
  DBuf<int32_t> wl_list;
  DBuf<unsigned long long> wl_cnt;
  DBuf<DedupEntry> dd_table;
  int64_t dd_mask = 0;
  DBuf<int64_t> dd_lead;
  int64_t dd_units = 0, dd_follow = 0;  // last call: units, followers (gvo_dedup_stats)
  bool dd_count = false;
  // work
  DBuf<int64_t> coefs;
  DBuf<int64_t> ctabs;
  DBuf<Geo> geos;
  DBuf<uint8_t> slab;
  int64_t run_cap = 16384, elem_cap = 1 << 19, slab_bytes = 0;
  int n_ctas = 0;
  DBuf<int> status;
  DBuf<unsigned long long> work;
  // key-range splitting state: header + queue + descriptor arena
  DBuf<uint8_t> split_mem;
  SplitState* split = nullptr;
  int64_t split_qcap = 1 << 22;
  int64_t sm_cap = 0;  // GVO_SMEM_ELEMS test hook
  int32_t seg_off = 0; // GVO_SEG=0 disables the segment cover (A/B hook)
  int32_t pat_off = 0; // GVO_PATTERN=0 disables pattern runs (A/B hook)
  int32_t wave_fm = 1;  // GVO_WAVE_ORDER=0: wave units config-major instead of field-major
  int32_t fuse_warp = 1; // GVO_FUSE_WARP=0: warp statistics as their own launch
  // Residency of the set kernel per batch: the 1-CTA/SM build (222 KB
  // bitmaps) wins on batches of multi-field LBM-like templates (C4), the
  // 2x320-thread build everywhere else (C2, C3, C5).  By default a batch of
  // >= 1024 configs takes sets1 when every registered template has >= 3
  // fields; GVO_BIG_BATCH=n forces sets1 for every batch of >= n configs.
  int64_t big_batch = 1024;
  bool big_forced = false;
  bool all_wide = false;     // every registered template has >= 3 fields
  bool any_wide = false;     // some registered template has >= 3 fields
  DBuf<int> wide_flag;       // per batch: 0 = every config's template has >= 3 fields
  int32_t epoch = 0;     // set-kernel launch counter (queue readiness tag)
  DBuf<uint8_t> rank_scratch;
  // host-variant staging
  DBuf<gvo_config> s_cfgs;
  DBuf<int64_t> s_counts, s_i64a, s_i64b, s_i64c, s_order;
  DBuf<double> s_stats, s_records, s_fd, s_gather;
  DBuf<int32_t> s_i32;
  DBuf<unsigned long long> s_ull;
  int64_t batch = 65536;  // configurations per device batch (GVO_BATCH, gvo_set_batch)
  // optional per-kernel timing (CUDA events on the launching stream)
  bool timing = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  double kernel_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t kernel_launches[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // optional per-unit statistics of the set engine (profiling)
  bool unit_debug = false;
  DBuf<int64_t> unit_stats;
  int64_t unit_items = 0;
};

// kernel ids for timing: 0 setup, 1 warp, 2 sets, 3 finish, 4 rank.  Every
// pipeline stage is also an NVTX range ("gvo.<stage>", nested in "gvo.batch"),
// so ncu --nvtx / any NVTX tool can attribute launches to stages.
struct NvtxRange {  // scoped: popped on every return path
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
static const char* const kStageName[5] = {"gvo.setup", "gvo.warp", "gvo.sets", "gvo.finish", "gvo.rank"};
static void tmark_begin(gvo_ctx* ctx, int id, cudaStream_t st, cudaEvent_t* b) {
  nvtxRangePushA(kStageName[id]);
  if (!ctx->timing) return;
  cudaEventCreate(b);
  cudaEventRecord(*b, st);
}
static void tmark_end(gvo_ctx* ctx, int id, cudaStream_t st, cudaEvent_t b) {
  nvtxRangePop();
  if (!ctx->timing) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  ctx->ev.push_back({id, {b, e}});
}

static int set_err(gvo_ctx* ctx, int code, const char* fmt, const char* detail = "") {
  if (ctx) {
    char buf[512];
    snprintf(buf, sizeof buf, fmt, detail);
    ctx->err = buf;
  }
  return code;
}
#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return set_err(ctx, GVO_ERR_CUDA, "CUDA error: %s", cudaGetErrorString(e_)); \
  } while (0)

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- translation classes (k_dedup.cu)
// Access `a` of field f is translation-safe when its value is exactly
// base_f + E(coordinates, block dims) with E free of every field base: the
// base enters through additions/subtractions only, with coefficient 1, never
// through *, // or % and no other field's base appears.  Moving base_f by Δ
// then moves every address of the field by Δ.
static bool base_additive(const gvo_insn* code, int len, int f) {
  int64_t st[64];
  int sp = 0;
  for (int i = 0; i < len; ++i) {
    const gvo_insn& in = code[i];
    if (in.op <= GVO_OP_BASE) {
      if (sp >= 64) return false;
      if (in.op == GVO_OP_BASE && in.arg != f) return false;
      st[sp++] = in.op == GVO_OP_BASE ? 1 : 0;
      continue;
    }
    if (sp < 2) return false;
    const int64_t r = st[--sp], l = st[--sp];
    int64_t o = 0;
    if (in.op == GVO_OP_ADD) o = l + r;
    else if (in.op == GVO_OP_SUB) o = l - r;
    else if (l != 0 || r != 0) return false;  // *, //, % of a base-carrying operand
    if (o < -8 || o > 8) return false;
    st[sp++] = o;
  }
  return sp == 1 && st[0] == 1;
}

static void put_bytes(std::string& k, const void* p, size_t n) { k.append(reinterpret_cast<const char*>(p), n); }

// fclass[field_base_off[t] + f] and tclass[t]: equal ids <=> the same
// accesses (kind, multiplicity, bytecode, in kernel order) up to the field
// bases, every access translation-safe; -1 = never shared
static void translation_classes(const gvo_template* t, int n, std::vector<int32_t>& fcls, std::vector<int32_t>& tcls) {
  std::unordered_map<std::string, int32_t> fmap, tmap;
  fcls.clear();
  tcls.assign(n, -1);
  for (int i = 0; i < n; ++i) {
    const gvo_template& T = t[i];
    bool all_ok = true;
    for (int f = 0; f < T.n_fields; ++f) {
      std::string key;
      bool ok = true;
      for (int a = 0; a < T.n_accesses && ok; ++a) {
        if (T.access_field[a] != f) continue;
        const gvo_insn* code = T.code + T.access_code_off[a];
        const int len = T.access_code_len[a];
        ok = base_additive(code, len, f);
        put_bytes(key, &T.access_kind[a], 4);
        put_bytes(key, &T.access_mult[a], 8);
        put_bytes(key, &len, 4);
        for (int k = 0; k < len; ++k) {
          put_bytes(key, &code[k].op, 4);
          const int64_t arg = code[k].op == GVO_OP_BASE ? -1 : code[k].arg;
          put_bytes(key, &arg, 8);
        }
      }
      int32_t id = -1;
      if (ok) {
        auto it = fmap.emplace(key, (int32_t)fmap.size()).first;
        id = it->second;
      }
      fcls.push_back(id);
      all_ok = all_ok && ok;
    }
    if (!all_ok) continue;
    std::string key;
    put_bytes(key, &T.n_fields, 4);
    for (int a = 0; a < T.n_accesses; ++a) {
      put_bytes(key, &T.access_field[a], 4);
      put_bytes(key, &T.access_kind[a], 4);
      put_bytes(key, &T.access_mult[a], 8);
      const int len = T.access_code_len[a];
      put_bytes(key, &len, 4);
      for (int k = 0; k < len; ++k) {
        const gvo_insn& in = T.code[T.access_code_off[a] + k];
        put_bytes(key, &in.op, 4);
        put_bytes(key, &in.arg, 8);
      }
    }
    tcls[i] = tmap.emplace(key, (int32_t)tmap.size()).first->second;
  }
}

extern "C" {

int gvo_abi_version(void) { return GVO_ABI_VERSION; }

int gvo_open(int device, gvo_ctx** out) {
  if (!out) return GVO_ERR_INVALID;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0) return GVO_ERR_CUDA;
  gvo_ctx* ctx = new gvo_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return GVO_ERR_CUDA; }
  cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return GVO_ERR_CUDA; }
  if (const char* e = getenv("GVO_ELEM_CAP")) ctx->elem_cap = atoll(e);
  if (const char* e = getenv("GVO_RUN_CAP")) ctx->run_cap = atoll(e);
  if (const char* e = getenv("GVO_BATCH")) ctx->batch = atoll(e);
  if (const char* e = getenv("GVO_SMEM_ELEMS")) ctx->sm_cap = atoll(e);
  if (const char* e = getenv("GVO_SEG")) ctx->seg_off = atoi(e) == 0;
  if (const char* e = getenv("GVO_PATTERN")) ctx->pat_off = atoi(e) == 0;
  if (const char* e = getenv("GVO_WAVE_ORDER")) ctx->wave_fm = atoi(e) != 0;
  if (const char* e = getenv("GVO_FUSE_WARP")) ctx->fuse_warp = atoi(e) != 0;
  if (const char* e = getenv("GVO_BIG_BATCH")) { ctx->big_batch = atoll(e); ctx->big_forced = true; }
  if (const char* e = getenv("GVO_DEDUP")) ctx->dedup = atoi(e) != 0;
  if (const char* e = getenv("GVO_PLAN_SHARE")) ctx->plan_share = atoi(e) != 0;
  if (const char* e = getenv("GVO_WORKLIST")) ctx->worklist = atoi(e) != 0;
  if (const char* e = getenv("GVO_HANDOFF_MIN")) ctx->handoff_min = atoll(e);
  ctx->n_ctas = kMaxSetsCtasPerSm * ctx->n_sm;
  *out = ctx;
  return GVO_OK;
}

void gvo_close(gvo_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto* b : {&ctx->t_nf, &ctx->t_na, &ctx->t_ab, &ctx->t_fbo, &ctx->t_af, &ctx->t_ak, &ctx->t_co,
                  &ctx->t_cl, &ctx->t_fko, &ctx->t_fkl, &ctx->s_i32})
    b->release();
  ctx->t_fb.release();
  ctx->t_am.release();
  ctx->t_fcls.release();
  ctx->t_tcls.release();
  ctx->d_mclass.release();
  ctx->dd_table.release();
  ctx->plan_table.release();
  ctx->plan_cache.release();
  ctx->plan_src.release();
  ctx->plan_used.release();
  ctx->plan_need.release();
  ctx->wl_list.release();
  ctx->wl_cnt.release();
  ctx->wide_flag.release();
  ctx->dd_lead.release();
  ctx->t_code.release();
  ctx->d_machines.release();
  ctx->coefs.release();
  ctx->ctabs.release();
  ctx->geos.release();
  ctx->work.release();
  ctx->s_order.release();
  ctx->unit_stats.release();
  ctx->slab.release();
  ctx->status.release();
  ctx->split_mem.release();
  ctx->rank_scratch.release();
  ctx->s_cfgs.release();
  ctx->s_counts.release();
  ctx->s_i64a.release();
  ctx->s_i64b.release();
  ctx->s_i64c.release();
  ctx->s_stats.release();
  ctx->s_records.release();
  ctx->s_fd.release();
  ctx->s_gather.release();
  ctx->s_ull.release();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (cudaEvent_t e : ctx->pipe_ev) cudaEventDestroy(e);
  delete ctx;
}

const char* gvo_last_error(const gvo_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gvo_set_templates(gvo_ctx* ctx, const gvo_template* t, int32_t n) {
  if (!ctx || !t || n <= 0) return set_err(ctx, GVO_ERR_INVALID, "invalid template list%s");
  CK(cudaSetDevice(ctx->device));
  std::vector<int32_t> nf(n), na(n), ab(n), fbo(n), af, ak, co, cl, fko, fkl;
  std::vector<int64_t> fb, am;
  std::vector<gvo_insn> code;
  int maxf = 0, maxa = 1;
  for (int i = 0; i < n; ++i) {
    const gvo_template& T = t[i];
    if (T.n_fields < 1 || T.n_fields > GVO_MAX_FIELDS)
      return set_err(ctx, GVO_ERR_UNSUPPORTED, "template has %s fields outside [1, 16]", std::to_string(T.n_fields).c_str());
    if (T.n_accesses < 1 || T.n_accesses > GVO_MAX_ACCESSES)
      return set_err(ctx, GVO_ERR_UNSUPPORTED, "template has %s accesses outside [1, 1024]", std::to_string(T.n_accesses).c_str());
    nf[i] = T.n_fields;
    na[i] = T.n_accesses;
    ab[i] = (int32_t)af.size();
    fbo[i] = (int32_t)fb.size();
    maxf = std::max(maxf, T.n_fields);
    maxa = std::max(maxa, T.n_accesses);
    for (int f = 0; f < T.n_fields; ++f) fb.push_back(T.field_base[f]);
    const int cbase = (int)code.size();
    for (int a = 0; a < T.n_accesses; ++a) {
      if (T.access_field[a] < 0 || T.access_field[a] >= T.n_fields || T.access_kind[a] < 0 || T.access_kind[a] > 1)
        return set_err(ctx, GVO_ERR_INVALID, "bad access descriptor%s");
      if (T.access_code_len[a] < 1 || T.access_code_len[a] > GVO_MAX_CODE)
        return set_err(ctx, GVO_ERR_UNSUPPORTED, "expression bytecode length outside [1, 256]%s");
      // stack depth check
      int sp = 0, mx = 0;
      for (int k = 0; k < T.access_code_len[a]; ++k) {
        const gvo_insn& in = T.code[T.access_code_off[a] + k];
        if (in.op <= GVO_OP_BASE) ++sp; else --sp;
        if (sp < 1) return set_err(ctx, GVO_ERR_INVALID, "malformed bytecode%s");
        mx = std::max(mx, sp);
        if ((in.op == GVO_OP_FLOORDIV || in.op == GVO_OP_MOD) &&
            (k == 0 || T.code[T.access_code_off[a] + k - 1].op != GVO_OP_CONST ||
             T.code[T.access_code_off[a] + k - 1].arg <= 0))
          return set_err(ctx, GVO_ERR_EXPR, "divisor of // and %% must be a positive constant%s");
      }
      if (sp != 1) return set_err(ctx, GVO_ERR_INVALID, "malformed bytecode%s");
      if (mx > kStack) return set_err(ctx, GVO_ERR_UNSUPPORTED, "expression deeper than 32 levels%s");
      af.push_back(T.access_field[a]);
      ak.push_back(T.access_kind[a]);
      am.push_back(T.access_mult[a]);
      co.push_back(cbase + T.access_code_off[a]);
      cl.push_back(T.access_code_len[a]);
    }
    for (int k = 0; k < T.n_code; ++k) code.push_back(T.code[k]);
    // (field, kind) access lists in kernel order
    const int fk0 = (int)fkl.size();
    for (int slot = 0; slot < 2 * GVO_MAX_FIELDS; ++slot) {
      fko.push_back((int32_t)(fkl.size() - fk0));
      for (int a = 0; a < T.n_accesses; ++a)
        if (T.access_field[a] * 2 + T.access_kind[a] == slot) fkl.push_back(a);
    }
    fko.push_back((int32_t)(fkl.size() - fk0));
    // make offsets absolute
    for (int slot = 0; slot <= 2 * GVO_MAX_FIELDS; ++slot) fko[fko.size() - 1 - slot] += fk0;
  }
  auto up32 = [&](DBuf<int32_t>& b, const std::vector<int32_t>& v) -> int {
    if (!b.ensure(std::max<size_t>(v.size(), 1))) return GVO_ERR_CUDA;
    if (!v.empty() && cudaMemcpy(b.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return GVO_ERR_CUDA;
    return GVO_OK;
  };
  auto up64 = [&](DBuf<int64_t>& b, const std::vector<int64_t>& v) -> int {
    if (!b.ensure(std::max<size_t>(v.size(), 1))) return GVO_ERR_CUDA;
    if (!v.empty() && cudaMemcpy(b.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return GVO_ERR_CUDA;
    return GVO_OK;
  };
  int rc = GVO_OK;
  rc |= up32(ctx->t_nf, nf); rc |= up32(ctx->t_na, na); rc |= up32(ctx->t_ab, ab); rc |= up32(ctx->t_fbo, fbo);
  rc |= up32(ctx->t_af, af); rc |= up32(ctx->t_ak, ak); rc |= up32(ctx->t_co, co); rc |= up32(ctx->t_cl, cl);
  rc |= up32(ctx->t_fko, fko); rc |= up32(ctx->t_fkl, fkl);
  rc |= up64(ctx->t_fb, fb); rc |= up64(ctx->t_am, am);
  {
    std::vector<int32_t> fcls, tcls;
    translation_classes(t, n, fcls, tcls);
    rc |= up32(ctx->t_fcls, fcls);
    rc |= up32(ctx->t_tcls, tcls);
  }
  if (rc) return set_err(ctx, GVO_ERR_CUDA, "template upload failed%s");
  if (!ctx->t_code.ensure(std::max<size_t>(code.size(), 1))) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpy(ctx->t_code.p, code.data(), code.size() * sizeof(gvo_insn), cudaMemcpyHostToDevice));
  ctx->n_tpl = n;
  ctx->max_fields = maxf;
  ctx->max_acc = maxa;
  ctx->h_nacc = na;
  ctx->h_nfields = nf;
  ctx->all_wide = !nf.empty();
  ctx->any_wide = false;
  for (int32_t f : nf) {
    ctx->all_wide = ctx->all_wide && f >= 3;
    ctx->any_wide = ctx->any_wide || f >= 3;
  }
  TplView& V = ctx->view;
  V.n_tpl = n;
  V.n_fields = ctx->t_nf.p; V.n_acc = ctx->t_na.p; V.acc_base = ctx->t_ab.p; V.field_base_off = ctx->t_fbo.p;
  V.field_base = ctx->t_fb.p; V.acc_field = ctx->t_af.p; V.acc_kind = ctx->t_ak.p; V.acc_mult = ctx->t_am.p;
  V.code_off = ctx->t_co.p; V.code_len = ctx->t_cl.p; V.code = ctx->t_code.p;
  V.fk_off = ctx->t_fko.p; V.fk_list = ctx->t_fkl.p; V.max_acc = maxa;
  V.fclass = ctx->t_fcls.p; V.tclass = ctx->t_tcls.p;
  // pageable cudaMemcpy may return before its DMA lands, and the pipeline
  // runs on non-blocking streams: make the upload visible to every stream
  CK(cudaDeviceSynchronize());
  return GVO_OK;
}

int gvo_set_machines(gvo_ctx* ctx, const gvo_machine* m, int32_t n) {
  if (!ctx || !m || n <= 0) return set_err(ctx, GVO_ERR_INVALID, "invalid machine list%s");
  CK(cudaSetDevice(ctx->device));
  for (int i = 0; i < n; ++i) {
    if (m[i].sector_bytes < 1 || m[i].l1_line_bytes % m[i].sector_bytes != 0 || m[i].l1_banks < 1 ||
        m[i].bank_width_bytes < 1 || m[i].sm_count < 1)
      return set_err(ctx, GVO_ERR_MACHINE, "invalid machine descriptor%s");
  }
  ctx->h_machines.assign(m, m + n);
  if (!ctx->d_machines.ensure(n)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpy(ctx->d_machines.p, m, n * sizeof(gvo_machine), cudaMemcpyHostToDevice));
  // machine classes: the integer parameters the set problems depend on
  // (granules, banks, waves); capacities, bandwidths, clock and fits only
  // enter the float assembly
  {
    std::vector<int32_t> mc(n);
    for (int i = 0; i < n; ++i) {
      mc[i] = i;
      for (int k = 0; k < i; ++k) {
        const gvo_machine &a = m[i], &b = m[k];
        if (a.sm_count == b.sm_count && a.l1_line_bytes == b.l1_line_bytes && a.sector_bytes == b.sector_bytes &&
            a.l1_banks == b.l1_banks && a.bank_width_bytes == b.bank_width_bytes &&
            a.max_threads_per_sm == b.max_threads_per_sm && a.max_blocks_per_sm == b.max_blocks_per_sm &&
            a.max_threads_per_block == b.max_threads_per_block) {
          mc[i] = mc[k];
          break;
        }
      }
    }
    if (!ctx->d_mclass.ensure(n)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
    CK(cudaMemcpy(ctx->d_mclass.p, mc.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  return GVO_OK;
}

static int ensure_work(gvo_ctx* ctx, int64_t n) {
  if (!ctx->coefs.ensure((size_t)n * ctx->max_acc * 8)) return set_err(ctx, GVO_ERR_CUDA, "coefficient table alloc failed%s");
  if (!ctx->geos.ensure((size_t)n)) return set_err(ctx, GVO_ERR_CUDA, "geometry alloc failed%s");
  if (!ctx->ctabs.ensure((size_t)n * ctab_stride(ctx->max_acc))) return set_err(ctx, GVO_ERR_CUDA, "class table alloc failed%s");
  if (ctx->slab_bytes == 0) {
    ctx->slab_bytes = sets_slab_bytes(ctx->run_cap, ctx->elem_cap);
    if (!ctx->slab.ensure((size_t)ctx->slab_bytes * ctx->n_ctas))
      return set_err(ctx, GVO_ERR_CUDA, "scratch slab alloc failed%s");
    // run records are copied whole (descriptor arena) although a run kind
    // leaves some fields unused: defined bytes for initcheck, once
    CK(cudaMemset(ctx->slab.p, 0, (size_t)ctx->slab_bytes * ctx->n_ctas));
  }
  // work[0] the set kernel's item counter, work[1] its block-unit pool, work[2..3] sharing statistics
  if (!ctx->status.ensure(4) || !ctx->work.ensure(4)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  if (!ctx->split) {
    const size_t hdr = 256;
    const size_t qb = (size_t)ctx->split_qcap * sizeof(RangeItem);
    const size_t n_slots = (size_t)ctx->n_ctas * kSplitSlotsPerCta;
    const size_t fb = (n_slots * sizeof(int32_t) + 255) & ~size_t(255);
    const size_t slot_bytes = split_slot_bytes(ctx->run_cap);
    if (!ctx->split_mem.ensure(hdr + qb + fb + n_slots * slot_bytes))
      return set_err(ctx, GVO_ERR_CUDA, "split alloc failed%s");
    SplitState h{};
    h.q_cap = ctx->split_qcap;
    h.arena_bytes = (int64_t)(n_slots * slot_bytes);
    h.queue = reinterpret_cast<RangeItem*>(ctx->split_mem.p + hdr);
    h.slot_busy = reinterpret_cast<int32_t*>(ctx->split_mem.p + hdr + qb);
    h.arena = ctx->split_mem.p + hdr + qb + fb;
    h.slot_bytes = (int64_t)slot_bytes;
    CK(cudaMemset(ctx->split_mem.p, 0, hdr + qb + fb));
    CK(cudaMemcpy(ctx->split_mem.p, &h, sizeof h, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    ctx->split = reinterpret_cast<SplitState*>(ctx->split_mem.p);
  }
  return GVO_OK;
}

static void sampling_eff(const gvo_sampling* s, int* S, int* W) {
  *S = std::min(std::max(s->block_samples, 1), GVO_MAX_BLOCK_SAMPLES);
  *W = std::min(std::max(s->wave_samples, 1), GVO_MAX_UNIQUE_WAVES - 1);
}

int64_t gvo_counts_stride_eff(int32_t F, const gvo_sampling* s) {
  int S, W;
  sampling_eff(s, &S, &W);
  return gvo_counts_stride(F, S, W);
}

int gvo_eval_configs(gvo_ctx* ctx, const gvo_config* d_cfgs, int64_t n, const gvo_sampling* sampling,
                     int32_t F, int64_t* d_counts, double* d_stats, double* d_records, double* d_field_down,
                     int64_t* d_l1_access, int32_t l1_stride, void* stream) {
  if (!ctx || !sampling || n < 0 || !d_counts || !d_records) return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  if (ctx->n_tpl == 0 || ctx->h_machines.empty()) return set_err(ctx, GVO_ERR_INVALID, "templates/machines not set%s");
  if (F < ctx->max_fields) return set_err(ctx, GVO_ERR_INVALID, "F smaller than the widest template%s");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = as_stream(stream);
  int S, W;
  sampling_eff(sampling, &S, &W);
  const int64_t stride = gvo_counts_stride(F, S, W);
  const gvo_machine& m0 = ctx->h_machines[0];
  // one sharing table per call (k_dedup.cu): keys of every batch, so later
  // batches reuse earlier batches' counts
  const bool dedup = ctx->dedup && n > 0 && ctx->t_fcls.p && ctx->d_mclass.p;
  if (dedup) {
    const int64_t want = 2 * dedup_units(n, F, S);
    int64_t cap = int64_t(1) << 12;
    while (cap < want && cap < (int64_t(1) << 23)) cap <<= 1;
    if (!ctx->dd_table.ensure((size_t)cap + 1) || !ctx->status.ensure(4))
      return set_err(ctx, GVO_ERR_CUDA, "sharing table alloc failed%s");
    ctx->dd_mask = cap - 1;
    CK(cudaMemsetAsync(ctx->dd_table.p, 0, (size_t)cap * sizeof(DedupEntry), st));
  }
  // plan sharing: one key table and leader-plan cache per call
  PlanShare PS{};
  if (ctx->plan_share && n > 1 && ctx->d_mclass.p) {
    int64_t cap = int64_t(1) << 10;
    while (cap < 2 * n && cap < (int64_t(1) << 22)) cap <<= 1;
    const int64_t words = plan_slot_words(ctx->max_acc);
    const int64_t slots = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(512) << 20) / (words * 8)));
    if (!ctx->plan_table.ensure((size_t)cap) || !ctx->plan_cache.ensure((size_t)(slots * words)) ||
        !ctx->plan_used.ensure(1) || !ctx->plan_src.ensure((size_t)std::min(n, ctx->batch)))
      return set_err(ctx, GVO_ERR_CUDA, "plan sharing alloc failed%s");
    CK(cudaMemsetAsync(ctx->plan_table.p, 0, (size_t)cap * sizeof(PlanEntry), st));
    CK(cudaMemsetAsync(ctx->plan_used.p, 0, sizeof(unsigned long long), st));
    PS.table = ctx->plan_table.p;
    PS.mask = cap - 1;
    PS.cache = ctx->plan_cache.p;
    PS.cap = slots;
    PS.n_used = ctx->plan_used.p;
    PS.src = ctx->plan_src.p;
    // followers' rows after the work lists, only where a unit computes
    if (ctx->worklist && ctx->plan_need.ensure((size_t)std::min(n, ctx->batch))) {
      PS.defer_rows = true;
      PS.need = ctx->plan_need.p;
    }
  }
  ctx->dd_units = ctx->dd_follow = 0;
  unsigned long long* dd_stats = nullptr;
  if (dedup && ctx->dd_count) {
    if (!ctx->work.ensure(4)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
    dd_stats = ctx->work.p + 2;
    CK(cudaMemsetAsync(dd_stats, 0, 2 * sizeof(unsigned long long), st));
  }
  for (int64_t b0 = 0; b0 < n; b0 += ctx->batch) {
    const int64_t nb = std::min(ctx->batch, n - b0);
    int rc = ensure_work(ctx, nb);
    if (rc) return rc;
    NvtxRange batch_range("gvo.batch");
    const gvo_config* cf = d_cfgs + b0;
    int64_t* cnt = d_counts + b0 * stride;
    CK(cudaMemsetAsync(cnt, 0, (size_t)nb * stride * 8, st));
    cudaEvent_t tb = nullptr;
    tmark_begin(ctx, 0, st, &tb);
    launch_setup(ctx->view, ctx->d_machines.p, cf, nb, *sampling, ctx->coefs.p, ctx->geos.p, ctx->ctabs.p, st,
                 ctx->d_mclass.p, PS.table ? &PS : nullptr);
    int64_t* lead = nullptr;
    if (dedup) {
      if (!ctx->dd_lead.ensure((size_t)dedup_units(nb, F, S))) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
      lead = ctx->dd_lead.p;
      launch_dedup(ctx->view, ctx->d_machines.p, ctx->d_mclass.p, cf, ctx->geos.p, nb, F, S, b0, ctx->dd_table.p,
                   ctx->dd_mask, lead, dd_stats, st);
    }
    tmark_end(ctx, 0, st, tb);
    // warp statistics: fused into the k_sets work queue when their shared
    // memory fits the set kernel's element buffer, else a separate launch
    WarpArgs WA{ctx->view, ctx->d_machines.p, cf, ctx->geos.p, ctx->coefs.p, nb * (S + 1), S, m0.sector_bytes,
               m0.bank_width_bytes, m0.l1_banks, 0, nullptr, cnt, stride, F,
               d_l1_access ? d_l1_access + b0 * l1_stride * 3 : nullptr, l1_stride, nullptr,
               lead ? lead + nb * F * (S + 1) : nullptr};
    const bool big = nb >= ctx->big_batch && (ctx->big_forced || ctx->all_wide);
    // mixed registries (e.g. C5: stencil and LBM templates): the residency is
    // chosen per batch on the device (every config's template has >= 3
    // fields -> the 1-CTA build), both launches queued, the other one exits
    const bool pick = !big && !ctx->big_forced && nb >= ctx->big_batch && ctx->any_wide;
    const bool fuse = ctx->fuse_warp &&
                      (int64_t)warp_item_smem(ctx->max_acc) <=
                          (big ? sets1::sets_ebuf_bytes()
                               : pick ? std::min(sets1::sets_ebuf_bytes(), sets2::sets_ebuf_bytes())
                                      : sets2::sets_ebuf_bytes());
    if (!fuse) {
      tmark_begin(ctx, 1, st, &tb);
      launch_warp(ctx->view, ctx->d_machines.p, cf, ctx->geos.p, ctx->coefs.p, nb * (S + 1), S, m0.sector_bytes,
                  m0.bank_width_bytes, m0.l1_banks, 0, nullptr, cnt, stride, F,
                  d_l1_access ? d_l1_access + b0 * l1_stride * 3 : nullptr, l1_stride, nullptr,
                  ctx->max_acc, ctx->n_sm, st);
      tmark_end(ctx, 1, st, tb);
    }
    SetsLaunch L{};
    L.T = ctx->view;
    L.machines = ctx->d_machines.p;
    L.cfgs = cf;
    L.geos = ctx->geos.p;
    L.coefs = ctx->coefs.p;
    L.ctabs = ctx->ctabs.p;
    L.n_items = nb * F * (S + 1);
    L.S_req = S;
    L.F_stride = F;
    L.mode = 0;
    L.counts = cnt;
    L.counts_stride = stride;
    L.slab = ctx->slab.p;
    L.slab_bytes = ctx->slab_bytes;
    L.run_cap = ctx->run_cap;
    L.elem_cap = ctx->elem_cap;
    L.status_out = ctx->status.p;
    L.n_ctas = ctx->n_ctas;
    L.work = ctx->work.p;
    L.split = ctx->split;
    L.sm_cap = ctx->sm_cap;
    L.seg_off = ctx->seg_off;
    L.pat_off = ctx->pat_off;
    L.wave_field_major = ctx->wave_fm;
    L.lead = lead;
    L.handoff = nb >= ctx->handoff_min ? 1 : 0;
    if (ctx->worklist && S > 0) {
      if (!ctx->wl_list.ensure((size_t)dedup_units(nb, F, S)) || !ctx->wl_cnt.ensure(3))
        return set_err(ctx, GVO_ERR_CUDA, "work list alloc failed%s");
      launch_worklists(ctx->view, cf, ctx->geos.p, nb, F, S, lead, ctx->wave_fm ? 1 : 0, ctx->wl_list.p,
                       ctx->wl_cnt.p, &L.wl_wave, &L.wl_blk, &L.wl_warp, PS.defer_rows ? ctx->plan_need.p : nullptr,
                       st);
      L.wl_cnt = ctx->wl_cnt.p;
    }
    if (PS.defer_rows) {
      tmark_begin(ctx, 0, st, &tb);
      launch_plan_rows(ctx->view, ctx->d_machines.p, cf, nb, *sampling, ctx->coefs.p, ctx->geos.p, ctx->ctabs.p, PS,
                       st);
      tmark_end(ctx, 0, st, tb);
    }
    if (fuse) {
      L.warp = WA;
      L.n_warp_items = WA.n_items;
    }
    if (ctx->unit_debug) {
      if (!ctx->unit_stats.ensure((size_t)L.n_items * 10 + 10 + 4096 * 10 + 1024 * 16)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
      CK(cudaMemsetAsync(ctx->unit_stats.p, 0, ((size_t)L.n_items * 10 + 10 + 4096 * 10 + 1024 * 16) * 8, st));
      L.unit_stats = ctx->unit_stats.p;
      ctx->unit_items = L.n_items;
    }
    tmark_begin(ctx, 2, st, &tb);
    if (++ctx->epoch == 0) ++ctx->epoch;
    L.epoch = ctx->epoch;
    if (big) {
      L.n_ctas = ctx->n_sm;
      sets1::launch_sets(L, st);
    } else if (pick) {
      if (!ctx->wide_flag.ensure(1)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
      launch_batch_wide(ctx->view, cf, nb, ctx->wide_flag.p, st);
      SetsLaunch L1 = L;
      L1.n_ctas = ctx->n_sm;
      L1.run_if = ctx->wide_flag.p;
      L1.run_if_val = 0;
      sets1::launch_sets(L1, st);
      if (++ctx->epoch == 0) ++ctx->epoch;
      L.epoch = ctx->epoch;
      L.run_if = ctx->wide_flag.p;
      L.run_if_val = 1;
      sets2::launch_sets(L, st);
    } else {
      sets2::launch_sets(L, st);
    }
    if (lead)
      launch_dedup_copy(cf, ctx->geos.p, ctx->view, d_counts, stride, nb, F, S, b0, lead, d_l1_access, l1_stride, st);
    tmark_end(ctx, 2, st, tb);
    tmark_begin(ctx, 3, st, &tb);
    launch_finish(ctx->view, ctx->d_machines.p, cf, ctx->geos.p, nb, S, W, F, cnt, stride,
                  d_stats ? d_stats + b0 * GVO_STATS_LEN(F) : nullptr, d_records + b0 * GVO_RECORD_LEN,
                  d_field_down ? d_field_down + b0 * 4 * F : nullptr, st);
    tmark_end(ctx, 3, st, tb);
    CK(cudaGetLastError());
    if (ctx->pipe.on) {  // this batch's rows are final: copy them out behind the next batches
      const size_t bi = (size_t)(b0 / ctx->batch);
      while (ctx->pipe_ev.size() <= bi) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->pipe_ev.push_back(e);
      }
      cudaStream_t cs = ctx->copy_stream;
      CK(cudaEventRecord(ctx->pipe_ev[bi], st));
      CK(cudaStreamWaitEvent(cs, ctx->pipe_ev[bi], 0));
      const auto& po = ctx->pipe;
      CK(cudaMemcpyAsync(po.counts + b0 * stride, cnt, (size_t)nb * stride * 8, cudaMemcpyDeviceToHost, cs));
      CK(cudaMemcpyAsync(po.records + b0 * GVO_RECORD_LEN, d_records + b0 * GVO_RECORD_LEN,
                         (size_t)nb * GVO_RECORD_LEN * 8, cudaMemcpyDeviceToHost, cs));
      if (po.stats && d_stats)
        CK(cudaMemcpyAsync(po.stats + b0 * GVO_STATS_LEN(F), d_stats + b0 * GVO_STATS_LEN(F),
                           (size_t)nb * GVO_STATS_LEN(F) * 8, cudaMemcpyDeviceToHost, cs));
      if (po.fd && d_field_down)
        CK(cudaMemcpyAsync(po.fd + b0 * 4 * F, d_field_down + b0 * 4 * F, (size_t)nb * 4 * F * 8,
                           cudaMemcpyDeviceToHost, cs));
      if (po.l1 && d_l1_access)
        CK(cudaMemcpyAsync(po.l1 + b0 * po.l1_stride * 3, d_l1_access + b0 * l1_stride * 3,
                           (size_t)nb * l1_stride * 3 * 8, cudaMemcpyDeviceToHost, cs));
    }
  }
  if (dd_stats) {
    unsigned long long h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, dd_stats, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->dd_units = (int64_t)h[0];
    ctx->dd_follow = (int64_t)h[1];
  }
  return GVO_OK;
}

int gvo_dedup_stats(gvo_ctx* ctx, int enable_counting, int64_t* shareable_units, int64_t* followers) {
  if (!ctx) return GVO_ERR_INVALID;
  ctx->dd_count = enable_counting != 0;
  if (shareable_units) *shareable_units = ctx->dd_units;
  if (followers) *followers = ctx->dd_follow;
  return ctx->dedup ? 1 : 0;
}

int gvo_set_batch(gvo_ctx* ctx, int64_t configs_per_batch) {
  if (!ctx || configs_per_batch < 1) return GVO_ERR_INVALID;
  ctx->batch = configs_per_batch;
  return GVO_OK;
}

int gvo_set_dedup(gvo_ctx* ctx, int enable) {
  if (!ctx) return GVO_ERR_INVALID;
  ctx->dedup = enable != 0;
  ctx->plan_share = enable != 0;
  return GVO_OK;
}

// Host-buffer entries: with page-locked outputs every batch's finished rows
// are copied out on a second stream behind the next batches' kernels.
// Returns 1 when the pipe is on (outputs then need no copy after the call).
static int pipe_begin(gvo_ctx* ctx, int64_t n, int64_t* h_counts, double* h_stats, double* h_records,
                      double* h_field_down, int64_t* h_l1_access, int32_t l1_stride) {
  auto pinned = [](const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost;
  };
  const bool pipe = n > ctx->batch && pinned(h_counts) && pinned(h_records) && pinned(h_stats) &&
                    pinned(h_field_down) && pinned(h_l1_access);
  if (!pipe) return 0;
  if (!ctx->copy_stream && cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  ctx->pipe.on = true;
  ctx->pipe.counts = h_counts;
  ctx->pipe.stats = h_stats;
  ctx->pipe.records = h_records;
  ctx->pipe.fd = h_field_down;
  ctx->pipe.l1 = h_l1_access;
  ctx->pipe.l1_stride = l1_stride;
  return 1;
}

int gvo_eval_configs_host(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n, const gvo_sampling* sampling,
                          int32_t F, int64_t* h_counts, double* h_stats, double* h_records,
                          double* h_field_down, int64_t* h_l1_access, int32_t l1_stride) {
  if (!ctx || !sampling || !h_cfgs || !h_counts || !h_records || n < 0)
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  int S, W;
  sampling_eff(sampling, &S, &W);
  const int64_t stride = gvo_counts_stride(F, S, W);
  cudaStream_t st = ctx->stream;
  if (!ctx->s_cfgs.ensure(std::max<int64_t>(n, 1)) || !ctx->s_counts.ensure(std::max<int64_t>(n * stride, 1)) ||
      !ctx->s_records.ensure(std::max<int64_t>(n * GVO_RECORD_LEN, 1)) ||
      (h_stats && !ctx->s_stats.ensure(std::max<int64_t>(n * GVO_STATS_LEN(F), 1))) ||
      (h_field_down && !ctx->s_fd.ensure(std::max<int64_t>(n * 4 * F, 1))) ||
      (h_l1_access && !ctx->s_i64a.ensure(std::max<int64_t>(n * l1_stride * 3, 1))))
    return set_err(ctx, GVO_ERR_CUDA, "staging alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_cfgs.p, h_cfgs, n * sizeof(gvo_config), cudaMemcpyHostToDevice, st));
  const int pipe = pipe_begin(ctx, n, h_counts, h_stats, h_records, h_field_down, h_l1_access, l1_stride);
  int rc = gvo_eval_configs(ctx, ctx->s_cfgs.p, n, sampling, F, ctx->s_counts.p,
                            h_stats ? ctx->s_stats.p : nullptr, ctx->s_records.p,
                            h_field_down ? ctx->s_fd.p : nullptr, h_l1_access ? ctx->s_i64a.p : nullptr,
                            l1_stride, st);
  ctx->pipe.on = false;
  if (pipe) CK(cudaStreamSynchronize(ctx->copy_stream));
  if (rc) return rc;
  if (!pipe) {
    CK(cudaMemcpyAsync(h_counts, ctx->s_counts.p, n * stride * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_records, ctx->s_records.p, n * GVO_RECORD_LEN * 8, cudaMemcpyDeviceToHost, st));
    if (h_stats) CK(cudaMemcpyAsync(h_stats, ctx->s_stats.p, n * GVO_STATS_LEN(F) * 8, cudaMemcpyDeviceToHost, st));
    if (h_field_down) CK(cudaMemcpyAsync(h_field_down, ctx->s_fd.p, n * 4 * F * 8, cudaMemcpyDeviceToHost, st));
    if (h_l1_access)
      CK(cudaMemcpyAsync(h_l1_access, ctx->s_i64a.p, n * l1_stride * 3 * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return GVO_OK;
}

int gvo_sweep_host_ex(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n, const gvo_sampling* sampling, int32_t F,
                      int64_t* h_counts, double* h_stats, double* h_records, double* h_field_down,
                      int64_t* h_l1_access, int32_t l1_stride, int64_t* h_order) {
  if (!ctx || !sampling || !h_cfgs || !h_counts || !h_records || !h_order || n < 0 || (h_l1_access && l1_stride < 1))
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  int S, W;
  sampling_eff(sampling, &S, &W);
  const int64_t stride = gvo_counts_stride(F, S, W);
  cudaStream_t st = ctx->stream;
  if (!ctx->s_cfgs.ensure(std::max<int64_t>(n, 1)) || !ctx->s_counts.ensure(std::max<int64_t>(n * stride, 1)) ||
      !ctx->s_records.ensure(std::max<int64_t>(n * GVO_RECORD_LEN, 1)) ||
      (h_stats && !ctx->s_stats.ensure(std::max<int64_t>(n * GVO_STATS_LEN(F), 1))) ||
      (h_field_down && !ctx->s_fd.ensure(std::max<int64_t>(n * 4 * F, 1))) ||
      (h_l1_access && !ctx->s_i64a.ensure(std::max<int64_t>(n * l1_stride * 3, 1))) ||
      !ctx->s_order.ensure(std::max<int64_t>(n, 1)))
    return set_err(ctx, GVO_ERR_CUDA, "staging alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_cfgs.p, h_cfgs, n * sizeof(gvo_config), cudaMemcpyHostToDevice, st));
  // page-locked outputs: copy each batch out while the next ones compute
  const int pipe = pipe_begin(ctx, n, h_counts, h_stats, h_records, h_field_down, h_l1_access, l1_stride);
  int rc = gvo_eval_configs(ctx, ctx->s_cfgs.p, n, sampling, F, ctx->s_counts.p, h_stats ? ctx->s_stats.p : nullptr,
                            ctx->s_records.p, h_field_down ? ctx->s_fd.p : nullptr,
                            h_l1_access ? ctx->s_i64a.p : nullptr, l1_stride, st);
  ctx->pipe.on = false;
  if (rc) {
    if (pipe) cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  rc = gvo_rank(ctx, ctx->s_records.p, ctx->s_cfgs.p, n, ctx->s_order.p, st);
  if (rc) {
    if (pipe) cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  if (!pipe) {
    CK(cudaMemcpyAsync(h_counts, ctx->s_counts.p, n * stride * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_records, ctx->s_records.p, n * GVO_RECORD_LEN * 8, cudaMemcpyDeviceToHost, st));
    if (h_stats) CK(cudaMemcpyAsync(h_stats, ctx->s_stats.p, n * GVO_STATS_LEN(F) * 8, cudaMemcpyDeviceToHost, st));
    if (h_field_down) CK(cudaMemcpyAsync(h_field_down, ctx->s_fd.p, n * 4 * F * 8, cudaMemcpyDeviceToHost, st));
    if (h_l1_access)
      CK(cudaMemcpyAsync(h_l1_access, ctx->s_i64a.p, n * l1_stride * 3 * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemcpyAsync(h_order, ctx->s_order.p, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (pipe) CK(cudaStreamSynchronize(ctx->copy_stream));
  return GVO_OK;
}

int gvo_sweep_host(gvo_ctx* ctx, const gvo_config* h_cfgs, int64_t n, const gvo_sampling* sampling, int32_t F,
                   int64_t* h_counts, double* h_stats, double* h_records, int64_t* h_order) {
  return gvo_sweep_host_ex(ctx, h_cfgs, n, sampling, F, h_counts, h_stats, h_records, nullptr, nullptr, 0, h_order);
}

int gvo_rank(gvo_ctx* ctx, const double* d_records, const gvo_config* d_cfgs, int64_t n, int64_t* d_order,
             void* stream) {
  if (!ctx || n < 0) return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->rank_scratch.ensure(rank_scratch_bytes(std::max<int64_t>(n, 1))))
    return set_err(ctx, GVO_ERR_CUDA, "rank scratch alloc failed%s");
  cudaEvent_t tb = nullptr;
  tmark_begin(ctx, 4, as_stream(stream), &tb);
  launch_rank(d_records, d_cfgs, n, d_order, ctx->rank_scratch.p, as_stream(stream));
  tmark_end(ctx, 4, as_stream(stream), tb);
  CK(cudaGetLastError());
  return GVO_OK;
}

int gvo_rank_gathered(gvo_ctx* ctx, const double* d_rows, const int64_t* d_gidx, int64_t n_rows,
                      const gvo_config* d_cfgs, int64_t n_global, double* d_records_global, int64_t* d_order,
                      void* stream) {
  if (!ctx || n_rows < 0 || n_global < 0 || (n_rows && (!d_rows || !d_gidx)) || (n_global && (!d_cfgs || !d_order)))
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = as_stream(stream);
  double* out = d_records_global;
  if (!out) {
    if (!ctx->s_gather.ensure(std::max<int64_t>(n_global * GVO_RECORD_LEN, 1)))
      return set_err(ctx, GVO_ERR_CUDA, "gather scratch alloc failed%s");
    out = ctx->s_gather.p;
  }
  if (!ctx->status.ensure(4)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  unsigned int* bad = reinterpret_cast<unsigned int*>(ctx->status.p + 3);
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned int), st));
  launch_scatter_gathered(d_rows, d_gidx, n_rows, n_global, out, bad, st);
  CK(cudaGetLastError());
  unsigned int h_bad = 0;
  CK(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h_bad) return set_err(ctx, GVO_ERR_INVALID, "gathered global index out of range%s");
  return gvo_rank(ctx, out, d_cfgs, n_global, d_order, stream);
}

const char* gvo_build_id(void) {
#ifdef GVO_BUILD_ID
  return GVO_BUILD_ID;
#else
  return "unknown";
#endif
}

// --------------------------------------------------------------- custom groups
static int one_config(gvo_ctx* ctx, int32_t tpl, const int32_t block[3], const int64_t grid[3]) {
  if (tpl < 0 || tpl >= ctx->n_tpl) return set_err(ctx, GVO_ERR_INVALID, "template id out of range%s");
  gvo_config c{};
  c.template_id = tpl;
  c.machine_id = 0;
  for (int k = 0; k < 3; ++k) { c.block[k] = block[k]; c.grid[k] = grid[k]; }
  c.work_per_thread = 1;
  int rc = ensure_work(ctx, 1);
  if (rc) return rc;
  if (!ctx->s_cfgs.ensure(1)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_cfgs.p, &c, sizeof c, cudaMemcpyHostToDevice, ctx->stream));
  k_coefs_only<<<1, 32, 0, ctx->stream>>>(ctx->view, ctx->s_cfgs.p, 1, ctx->coefs.p);
  launch_classes(ctx->view, ctx->s_cfgs.p, 1, ctx->coefs.p, ctx->ctabs.p, ctx->stream);
  CK(cudaGetLastError());
  return GVO_OK;
}

int gvo_group_footprint(gvo_ctx* ctx, int32_t tpl, const int32_t block[3], const int64_t grid[3],
                        const int64_t* h_run_start, const int64_t* h_run_count, int32_t n_runs,
                        int64_t granularity, int64_t* h_out) {
  if (!ctx || !h_out || n_runs < 1 || granularity < 1) return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  int rc = one_config(ctx, tpl, block, grid);
  if (rc) return rc;
  const int F = ctx->h_nfields[tpl];
  cudaStream_t st = ctx->stream;
  // host geometry: tpb only
  Geo G{};
  G.status = GVO_OK;
  G.phases = 7;
  G.tpb = (int64_t)block[0] * block[1] * block[2];
  G.lups_per_block = G.tpb;
  CK(cudaMemcpyAsync(ctx->geos.p, &G, sizeof G, cudaMemcpyHostToDevice, st));
  std::vector<int64_t> blocks;
  for (int r = 0; r < n_runs; ++r)
    for (int64_t b = 0; b < h_run_count[r]; ++b) blocks.push_back(h_run_start[r] + b);
  if (!ctx->s_i64a.ensure(n_runs) || !ctx->s_i64b.ensure(n_runs) || !ctx->s_i64c.ensure(std::max<size_t>(blocks.size(), 1)) ||
      !ctx->s_counts.ensure(2 * GVO_MAX_FIELDS) || !ctx->s_ull.ensure(2 * GVO_MAX_FIELDS))
    return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_i64a.p, h_run_start, n_runs * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_i64b.p, h_run_count, n_runs * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_i64c.p, blocks.data(), blocks.size() * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->s_counts.p, 0, 2 * GVO_MAX_FIELDS * 8, st));
  CK(cudaMemsetAsync(ctx->s_ull.p, 0, 2 * GVO_MAX_FIELDS * 8, st));
  CK(cudaMemsetAsync(ctx->status.p, 0, 4, st));
  SetsLaunch L{};
  L.T = ctx->view;
  L.machines = ctx->d_machines.p;
  L.cfgs = ctx->s_cfgs.p;
  L.geos = ctx->geos.p;
  L.coefs = ctx->coefs.p;
  L.ctabs = ctx->ctabs.p;
  L.n_items = F;
  L.S_req = 0;
  L.F_stride = F;
  L.mode = 2;
  L.granularity = granularity;
  L.run_start = ctx->s_i64a.p;
  L.run_count = ctx->s_i64b.p;
  L.n_custom_runs = n_runs;
  L.counts = ctx->s_counts.p;
  L.counts_stride = 0;
  L.slab = ctx->slab.p;
  L.slab_bytes = ctx->slab_bytes;
  L.run_cap = ctx->run_cap;
  L.elem_cap = ctx->elem_cap;
  L.status_out = ctx->status.p;
  L.n_ctas = ctx->n_ctas;
  L.work = ctx->work.p;
  L.split = ctx->split;
    L.sm_cap = ctx->sm_cap;
    L.seg_off = ctx->seg_off;
    L.pat_off = ctx->pat_off;
    L.wave_field_major = ctx->wave_fm;
  if (++ctx->epoch == 0) ++ctx->epoch;
  L.epoch = ctx->epoch;
  sets2::launch_sets(L, st);
  launch_warp(ctx->view, ctx->d_machines.p, ctx->s_cfgs.p, ctx->geos.p, ctx->coefs.p, (int64_t)blocks.size(), 0, granularity, 1, 1, 1,
              ctx->s_i64c.p, nullptr, 0, F, nullptr, 0, ctx->s_ull.p, ctx->max_acc, ctx->n_sm, st);
  CK(cudaGetLastError());
  int64_t uniq[2 * GVO_MAX_FIELDS];
  unsigned long long tot[2 * GVO_MAX_FIELDS];
  int status = 0;
  CK(cudaMemcpyAsync(uniq, ctx->s_counts.p, sizeof uniq, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(tot, ctx->s_ull.p, sizeof tot, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&status, ctx->status.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (status) return set_err(ctx, status, "group footprint engine status %s", std::to_string(status).c_str());
  for (int f = 0; f < F; ++f)
    for (int k = 0; k < 2; ++k) {
      h_out[(f * 2 + k) * 2 + 0] = uniq[f * 2 + k];
      h_out[(f * 2 + k) * 2 + 1] = (int64_t)tot[f * 2 + k];
    }
  return GVO_OK;
}

int gvo_group_sets(gvo_ctx* ctx, int32_t tpl, const int32_t block[3], const int64_t grid[3],
                   const int64_t* h_run_start, const int64_t* h_run_count, int32_t n_groups,
                   int64_t granularity, int64_t* h_out) {
  if (!ctx || !h_out || n_groups < 1 || n_groups > GVO_MAX_UNIQUE_WAVES || granularity < 1)
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  int rc = one_config(ctx, tpl, block, grid);
  if (rc) return rc;
  const int F = ctx->h_nfields[tpl];
  cudaStream_t st = ctx->stream;
  Geo G{};
  G.status = GVO_OK;
  G.phases = 7;
  G.tpb = (int64_t)block[0] * block[1] * block[2];
  G.lups_per_block = G.tpb;
  G.n_uw = n_groups;
  for (int u = 0; u < n_groups; ++u) { G.uw_start[u] = h_run_start[u]; G.uw_count[u] = h_run_count[u]; }
  CK(cudaMemcpyAsync(ctx->geos.p, &G, sizeof G, cudaMemcpyHostToDevice, st));
  const size_t nout = (size_t)n_groups * F * 4;
  if (!ctx->s_counts.ensure(nout)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemsetAsync(ctx->s_counts.p, 0, nout * 8, st));
  CK(cudaMemsetAsync(ctx->status.p, 0, 4, st));
  SetsLaunch L{};
  L.T = ctx->view;
  L.machines = ctx->d_machines.p;
  L.cfgs = ctx->s_cfgs.p;
  L.geos = ctx->geos.p;
  L.coefs = ctx->coefs.p;
  L.ctabs = ctx->ctabs.p;
  L.n_items = F;
  L.F_stride = F;
  L.mode = 1;
  L.granularity = granularity;
  L.counts = ctx->s_counts.p;
  L.slab = ctx->slab.p;
  L.slab_bytes = ctx->slab_bytes;
  L.run_cap = ctx->run_cap;
  L.elem_cap = ctx->elem_cap;
  L.status_out = ctx->status.p;
  L.n_ctas = ctx->n_ctas;
  L.work = ctx->work.p;
  L.split = ctx->split;
    L.sm_cap = ctx->sm_cap;
    L.seg_off = ctx->seg_off;
    L.pat_off = ctx->pat_off;
    L.wave_field_major = ctx->wave_fm;
  if (++ctx->epoch == 0) ++ctx->epoch;
  L.epoch = ctx->epoch;
  sets2::launch_sets(L, st);
  CK(cudaGetLastError());
  int status = 0;
  CK(cudaMemcpyAsync(h_out, ctx->s_counts.p, nout * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&status, ctx->status.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (status) return set_err(ctx, status, "group sets engine status %s", std::to_string(status).c_str());
  return GVO_OK;
}

int gvo_l1_cycles(gvo_ctx* ctx, int32_t tpl, const int32_t block[3], const int64_t grid[3], int64_t block_linear,
                  int64_t bank_width_bytes, int64_t n_banks, int64_t* h_out) {
  if (!ctx || !h_out || bank_width_bytes < 1 || n_banks < 1) return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  CK(cudaSetDevice(ctx->device));
  int rc = one_config(ctx, tpl, block, grid);
  if (rc) return rc;
  cudaStream_t st = ctx->stream;
  const int A = ctx->h_nacc[tpl];
  Geo G{};
  G.status = GVO_OK;
  G.phases = 7;
  G.tpb = (int64_t)block[0] * block[1] * block[2];
  CK(cudaMemcpyAsync(ctx->geos.p, &G, sizeof G, cudaMemcpyHostToDevice, st));
  if (!ctx->s_i64c.ensure(1) || !ctx->s_ull.ensure(3 * (size_t)A)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_i64c.p, &block_linear, 8, cudaMemcpyHostToDevice, st));
  launch_warp(ctx->view, ctx->d_machines.p, ctx->s_cfgs.p, ctx->geos.p, ctx->coefs.p, 1, 0, 1, bank_width_bytes, n_banks, 2,
              ctx->s_i64c.p, nullptr, 0, 0, nullptr, 0, ctx->s_ull.p, ctx->max_acc, ctx->n_sm, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_out, ctx->s_ull.p, 3 * (size_t)A * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return GVO_OK;
}

int gvo_eval_addresses(gvo_ctx* ctx, int32_t tpl, int32_t access, const int32_t block[3], const int64_t* h_coords,
                       int64_t n, int64_t* h_out) {
  if (!ctx || tpl < 0 || tpl >= ctx->n_tpl || access < 0 || access >= ctx->h_nacc[tpl] || n < 0)
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  if (n == 0) return GVO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (!ctx->s_i64a.ensure(n * 6) || !ctx->s_i64b.ensure(n)) return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_i64a.p, h_coords, n * 6 * 8, cudaMemcpyHostToDevice, st));
  k_eval_addresses<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctx->view, tpl, access, block[0], block[1], block[2],
                                                               ctx->s_i64a.p, n, ctx->s_i64b.p);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_out, ctx->s_i64b.p, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return GVO_OK;
}

int gvo_assemble_host(gvo_ctx* ctx, const double* h_stats, int32_t F, const int32_t* h_mid, const int64_t* h_flops,
                      int64_t n, double* h_records, double* h_field_down) {
  if (!ctx || !h_stats || !h_mid || !h_flops || !h_records || n < 0 || F < 1 || F > GVO_MAX_FIELDS)
    return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  if (n == 0) return GVO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (!ctx->s_stats.ensure(n * GVO_STATS_LEN(F)) || !ctx->s_i32.ensure(n) || !ctx->s_i64a.ensure(n) ||
      !ctx->s_records.ensure(n * GVO_RECORD_LEN) || !ctx->s_fd.ensure(n * 4 * F))
    return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_stats.p, h_stats, n * GVO_STATS_LEN(F) * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_i32.p, h_mid, n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_i64a.p, h_flops, n * 8, cudaMemcpyHostToDevice, st));
  launch_assemble_stats(ctx->d_machines.p, ctx->s_i32.p, ctx->s_i64a.p, n, F, ctx->s_stats.p, ctx->s_records.p,
                        h_field_down ? ctx->s_fd.p : nullptr, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_records, ctx->s_records.p, n * GVO_RECORD_LEN * 8, cudaMemcpyDeviceToHost, st));
  if (h_field_down) CK(cudaMemcpyAsync(h_field_down, ctx->s_fd.p, n * 4 * F * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return GVO_OK;
}

int gvo_set_timing(gvo_ctx* ctx, int enable) {
  if (!ctx) return GVO_ERR_INVALID;
  ctx->timing = enable != 0;
  return GVO_OK;
}

// Drains recorded events (synchronising on them) and returns accumulated
// per-kernel milliseconds and launch-group counts since the last reset.
int gvo_kernel_times(gvo_ctx* ctx, double* ms_out, int64_t* count_out, int reset) {
  if (!ctx) return GVO_ERR_INVALID;
  for (auto& x : ctx->ev) {
    cudaEventSynchronize(x.second.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, x.second.first, x.second.second);
    ctx->kernel_ms[x.first] += ms;
    ctx->kernel_launches[x.first] += 1;
    cudaEventDestroy(x.second.first);
    cudaEventDestroy(x.second.second);
  }
  ctx->ev.clear();
  for (int k = 0; k < 8; ++k) {
    if (ms_out) ms_out[k] = ctx->kernel_ms[k];
    if (count_out) count_out[k] = ctx->kernel_launches[k];
    if (reset) { ctx->kernel_ms[k] = 0; ctx->kernel_launches[k] = 0; }
  }
  return GVO_OK;
}

int gvo_debug_units(gvo_ctx* ctx, int enable, int64_t* h_out, int64_t cap, int64_t* n_items) {
  if (!ctx) return GVO_ERR_INVALID;
  ctx->unit_debug = enable != 0;
  if (n_items) *n_items = ctx->unit_items;
  if (h_out && ctx->unit_items) {
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h_out, ctx->unit_stats.p, std::min<int64_t>(cap, ctx->unit_items * 10 + 10 + 4096 * 10 + 1024 * 16) * 8, cudaMemcpyDeviceToHost));
  }
  return GVO_OK;
}

int gvo_int_peak(gvo_ctx* ctx, double* ops_per_s) {
  if (!ctx || !ops_per_s) return GVO_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  return launch_int_peak(ctx->n_sm, ctx->stream, ops_per_s) ? GVO_ERR_CUDA : GVO_OK;
}

int gvo_predict_host(gvo_ctx* ctx, const int32_t* h_mid, const double* h_dd, const double* h_ld,
                     const double* h_cyc, const int64_t* h_fl, int64_t n, double* h_out) {
  if (!ctx || n < 0) return set_err(ctx, GVO_ERR_INVALID, "invalid arguments%s");
  if (n == 0) return GVO_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (!ctx->s_i32.ensure(n) || !ctx->s_stats.ensure(3 * n) || !ctx->s_i64a.ensure(n) || !ctx->s_records.ensure(6 * n))
    return set_err(ctx, GVO_ERR_CUDA, "alloc failed%s");
  CK(cudaMemcpyAsync(ctx->s_i32.p, h_mid, n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_stats.p, h_dd, n * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_stats.p + n, h_ld, n * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_stats.p + 2 * n, h_cyc, n * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->s_i64a.p, h_fl, n * 8, cudaMemcpyHostToDevice, st));
  launch_predict(ctx->d_machines.p, ctx->s_i32.p, ctx->s_stats.p, ctx->s_stats.p + n, ctx->s_stats.p + 2 * n,
                 ctx->s_i64a.p, n, ctx->s_records.p, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h_out, ctx->s_records.p, n * 6 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return GVO_OK;
}

}  // extern "C"
