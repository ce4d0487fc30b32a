// vexsort_b200.cu -- host driver + C ABI (include/vexsort_b200.h).
//
// One translation unit: the kernels (partition2.cuh, bitonic.cuh,
// qsort.cuh) are instantiated here for the element kinds of the reference
// (int32, float64) and their same-width payloads (uint32 / uint64).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vexsort_b200.h"
#include "common.cuh"
#include "partition2.cuh"
#include "qsort.cuh"
#include "finish.cuh"
#include "scatter.cuh"
#include "hist.cuh"
#include "local.cuh"

using namespace vx;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define VX_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(VX_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define VX_LAUNCHED()                                                                        \
    do {                                                                                     \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess) return fail(VX_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// Opt a kernel into > 48 KB dynamic shared memory and return its resident
// CTAs per SM for that smem size.
template <typename F>
int prepare(F* kernel, int threads, size_t smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    return occ > 0 ? occ : 1;
}

// -------------------------------------------------------------- sort layout
template <typename K, typename V>
struct SortLayout {
    static constexpr uint32_t LOCAL = FinCap<K, V>::value;
    static constexpr int TILE = qs_tile<K>();
    uint64_t n = 0;
    uint64_t cap_seg = 0, cap_spl = 0, cap_bkt = 0, cap_tiles = 0, cap_fin = 0;
    size_t off_sk = 0, off_sv = 0, off_seg0 = 0, off_seg1 = 0, off_ctl = 0, off_spl = 0, off_bkt = 0,
           off_tile = 0, off_fin = 0, off_ids = 0, off_ql = 0, total = 0;

    explicit SortLayout(uint64_t n_) : n(n_) {
        constexpr bool KV = HasVal<V>::value;
        cap_seg = n / (LOCAL + 1) + 2;
        cap_spl = 2 * n / LOCAL + 2 * cap_seg + 512;
        cap_bkt = 2 * cap_spl + cap_seg;
        cap_tiles = n / TILE + cap_seg + 1;
        cap_fin = 2 * cap_bkt + n / kCopyChunk + 16;
        size_t o = 0;
        off_sk = o; o = align_up(o + n * sizeof(K));
        off_sv = o; o = align_up(o + (KV ? n * sizeof(V) : 0));
        off_seg0 = o; o = align_up(o + cap_seg * sizeof(Seg));
        off_seg1 = o; o = align_up(o + cap_seg * sizeof(Seg));
        off_ctl = o; o = align_up(o + kMaxLevels * sizeof(Ctl));
        off_spl = o; o = align_up(o + cap_spl * sizeof(K));
        off_bkt = o; o = align_up(o + cap_bkt * sizeof(unsigned long long));
        off_tile = o; o = align_up(o + cap_tiles * sizeof(unsigned));
        off_fin = o; o = align_up(o + 2 * cap_fin * sizeof(Fin));  // ping-pong by level parity
        off_ids = o; o = align_up(o + n * sizeof(unsigned short));  // per-element bucket ids (hist -> scatter)
        off_ql = o; o = align_up(o + cap_seg * sizeof(QlItemT));      // CTA-local level queue
        total = o;
    }
};

struct PinnedScratch {
    unsigned long long* p = nullptr;
    unsigned long long* get() {
        if (!p) cudaHostAlloc((void**)&p, 256, cudaHostAllocDefault);
        return p;
    }
};
thread_local PinnedScratch g_pinned;

// ----------------------------------------------------------- instrumentation
// Launch counting is always on; per-launch CUDA-event timing is opt-in
// (vx_profile_enable) and brackets each kernel on its own stream.
enum KClass { KC_PLAN = 0, KC_HIST, KC_EMIT, KC_SCATTER, KC_FINISH, KC_PARTITION, KC_SEGSORT, KC_BUCKET, KC_LOCAL,
              KC_N };
struct KProf {
    std::mutex mu;
    bool on = false;
    long long launches[KC_N] = {};
    double ms[KC_N] = {};
    unsigned long long elems[KC_N] = {};
    struct Pending { int cls; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t ev() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
KProf g_prof;

struct Launch {  // RAII bracket: count the launch, optionally time it
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    Launch(int c, cudaStream_t s, int count = 1) : cls(c), st(s) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.launches[cls] += count;
        if (g_prof.on) {
            a = g_prof.ev();
            b = g_prof.ev();
            cudaEventRecord(a, st);
        }
    }
    ~Launch() {
        if (a) {
            cudaEventRecord(b, st);
            std::lock_guard<std::mutex> lk(g_prof.mu);
            g_prof.pending.push_back({cls, a, b});
        }
    }
};

void prof_collect() {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (auto& p : g_prof.pending) {
        cudaEventSynchronize(p.b);
        float t = 0.f;
        if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) g_prof.ms[p.cls] += t;
        g_prof.pool.push_back(p.a);
        g_prof.pool.push_back(p.b);
    }
    g_prof.pending.clear();
}
void prof_elems(int cls, unsigned long long e) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.elems[cls] += e;
}

// in_k may equal out_k (in place).  Level 0 reads the input; every later
// level and the finish kernels work in out / scratch only, so an
// out-of-place sort leaves the input untouched at no extra traffic.
template <typename K, typename V>
int run_sort(const K* in_k, const V* in_v, K* keys, V* vals, uint64_t n, const vx_sort_config* cfg, void* ws,
             size_t ws_bytes, cudaStream_t st) {
    using L = SortLayout<K, V>;
    if (n < 2) {
        if (n == 1 && in_k != keys) {
            VX_CUDA(cudaMemcpyAsync(keys, in_k, sizeof(K), cudaMemcpyDeviceToDevice, st));
            if (HasVal<V>::value) VX_CUDA(cudaMemcpyAsync(vals, in_v, sizeof(V), cudaMemcpyDeviceToDevice, st));
        }
        return VX_OK;
    }
    L lay(n);
    if (ws_bytes < lay.total || !ws) return fail(VX_EWORKSPACE, "sort workspace too small");
    const int lanes = sizeof(K) == 4 ? 16 : 8;
    int64_t bound = cfg && cfg->sort_bound > 0 ? cfg->sort_bound : 16 * lanes;
    if (bound < 1 || bound > 16 * lanes) return fail(VX_EINVAL, "sort_bound exceeds small-sort capacity");
    const uint64_t seed = mix64(cfg ? cfg->pivot_seed : 0);

    char* w = static_cast<char*>(ws);
    K* sk = reinterpret_cast<K*>(w + lay.off_sk);
    V* sv = reinterpret_cast<V*>(w + lay.off_sv);
    Seg* segs[2] = {reinterpret_cast<Seg*>(w + lay.off_seg0), reinterpret_cast<Seg*>(w + lay.off_seg1)};
    Ctl* ctl = reinterpret_cast<Ctl*>(w + lay.off_ctl);
    K* spl = reinterpret_cast<K*>(w + lay.off_spl);
    unsigned long long* bkt = reinterpret_cast<unsigned long long*>(w + lay.off_bkt);
    unsigned* towner = reinterpret_cast<unsigned*>(w + lay.off_tile);
    Fin* fins[2] = {reinterpret_cast<Fin*>(w + lay.off_fin), reinterpret_cast<Fin*>(w + lay.off_fin) + lay.cap_fin};
    unsigned short* ids = reinterpret_cast<unsigned short*>(w + lay.off_ids);
    // the bitonic leaf bound: the reference's sort_bound when given, else
    // the widest warp network (512); see DESIGN.md
    const unsigned leaf = (cfg && cfg->sort_bound > 0) ? (unsigned)bound : kWarpSortMax;
    QlItemT* qls = reinterpret_cast<QlItemT*>(w + lay.off_ql);
#ifndef VX_NO_QL
    // the CTA-local level needs leaves of ~2x its bucket target (skipped for a
    // small sort_bound) and enough segments to fill the GPU (one CTA each):
    // below ~256 target-sized segments the finish path alone is faster
    const bool ql_on = leaf >= 2 * QlCfg<K, V>::LT && n >= 256 * QlCfg<K, V>::TARGET;
#else
    const bool ql_on = false;
#endif
    // leaves as small as the level count allows (L2 residency of the
    // CTA-local working set): the levels needed at the full target, then
    // the smallest target in [TMIN, TARGET] that needs no more of them
    uint64_t ql_target = 0;
    if (ql_on) {
        const double L = ceil(log((double)n / (double)QlCfg<K, V>::TARGET) / log(256.0) - 1e-9);
        const double t = (double)n / pow(256.0, L < 1.0 ? 1.0 : L);
        ql_target = (uint64_t)std::min((double)QlCfg<K, V>::TARGET, std::max((double)QlCfg<K, V>::TMIN, ceil(t)));
    }
    const uint64_t ql_cap = ql_on ? QlCfg<K, V>::CAP : 0;
    if (!HasVal<V>::value) sv = nullptr;

    const int sms = num_sms();
    static int occ_hist = prepare(qs_hist_kernel<K>, kQsNT, hist_smem_bytes<K>());
    static int occ_scat = prepare(qs_scatter_kernel<K, V>, kQsNT, sizeof(ScatterPipeSmem<K, V>));
    static int occ_fin = prepare(qs_finish_kernel<K, V>, kFinNT, sizeof(FinSmem<K, V>));
    static int occ_loc = prepare(qs_local_kernel<K, V>, kQlNT, sizeof(QlSmem<K, V>));
    const int g_hist = sms * occ_hist, g_scat = sms * occ_scat, g_fin = sms * occ_fin;

    VX_CUDA(cudaMemsetAsync(ctl, 0, kMaxLevels * sizeof(Ctl), st));
    unsigned long long* hp = g_pinned.get();
    if (!hp) return fail(VX_ECUDA, "cudaHostAlloc failed");
    unsigned nseg = 0;
    const K* root_scr_k = sk;
    const V* root_scr_v = sv;
    if (n <= L::LOCAL) {
        // the whole array is one finish item; its source is the input
        Fin f{0ull, (unsigned)n, in_k == keys ? 0u : 1u};
        VX_CUDA(cudaMemcpyAsync(fins[0], &f, sizeof(Fin), cudaMemcpyHostToDevice, st));
        unsigned one = 1;
        VX_CUDA(cudaMemcpyAsync(&ctl[0].fin_ctr, &one, sizeof(unsigned), cudaMemcpyHostToDevice, st));
        root_scr_k = in_k;
        root_scr_v = in_v;
    } else {
        qs_init_kernel<<<1, 1, 0, st>>>(segs[0], ctl, n);
        VX_LAUNCHED();
        nseg = 1;
    }
    for (int level = 0; level < kMaxLevels - 1; ++level) {
        const bool even = (level & 1) == 0;
        Ctl* c = ctl + level;
        const uint64_t lvl_seed = mix64(seed + 0x51ED270B27AD1CULL * (level + 1));
        if (nseg > 0) {
            const K* src_k = level == 0 ? in_k : (even ? keys : sk);
            const V* src_v = level == 0 ? in_v : (even ? vals : sv);
            K* dst_k = even ? sk : keys;
            V* dst_v = even ? sv : vals;
            const unsigned g_seg = std::min<unsigned>(nseg, (unsigned)sms * 4);
            {
                Launch l(KC_PLAN, st);
                qs_plan_kernel<K, V><<<g_seg, kPlanNT, 0, st>>>(src_k, segs[level & 1], c, spl, bkt, towner,
                                                                 (unsigned)lay.cap_spl, (unsigned)lay.cap_bkt,
                                                                 (unsigned)lay.cap_tiles, lvl_seed, ql_target);
            }
            VX_LAUNCHED();
            {
                Launch l(KC_HIST, st);
                qs_hist_kernel<K><<<g_hist, kQsNT, hist_smem_bytes<K>(), st>>>(src_k, n, segs[level & 1], c, towner,
                                                                                spl, bkt, ids);
            }
            VX_LAUNCHED();
            {
                Launch l(KC_EMIT, st);
                qs_emit_kernel<K, V><<<g_seg, kPlanNT, 0, st>>>(segs[level & 1], c, ctl + level + 1,
                                                                 segs[(level + 1) & 1], bkt, fins[level & 1],
                                                                 (unsigned)lay.cap_seg, (unsigned)lay.cap_fin,
                                                                 even ? 1 : 0, spl, qls, ql_cap);
            }
            VX_LAUNCHED();
            {
                Launch l(KC_SCATTER, st);
                qs_scatter_kernel<K, V><<<g_scat, kQsNT, sizeof(ScatterPipeSmem<K, V>), st>>>(
                    src_k, src_v, ids, dst_k, dst_v, segs[level & 1], c, towner, bkt);
            }
            VX_LAUNCHED();
            if (ql_cap) {
                // medium children: CTA-local last level + leaves (data in dst, other buffer = src side)
                Launch l(KC_LOCAL, st);
                qs_local_kernel<K, V><<<sms * occ_loc, kQlNT, sizeof(QlSmem<K, V>), st>>>(
                    qls, c, ctl + level + 1, segs[(level + 1) & 1], (unsigned)lay.cap_seg, dst_k, dst_v,
                    even ? keys : sk, even ? vals : sv, keys, vals, leaf);
            }
            VX_LAUNCHED();
        }
        {
            Launch l(KC_FINISH, st);
            const K* scr_k = level == 0 ? root_scr_k : sk;
            const V* scr_v = level == 0 ? root_scr_v : sv;
            qs_finish_kernel<K, V><<<g_fin, kFinNT, sizeof(FinSmem<K, V>), st>>>(
                fins[level & 1], c, ctl + level + 1, fins[(level + 1) & 1], (unsigned)lay.cap_fin, keys, vals, scr_k,
                scr_v, lvl_seed, leaf);
        }
        VX_LAUNCHED();
        // this level's error flag and element counters and the next level's
        // queue sizes -> host: the two adjacent Ctl records in one copy
        static_assert(2 * sizeof(Ctl) <= 256, "pinned scratch holds two Ctl records");
        Ctl* hc = reinterpret_cast<Ctl*>(hp);
        VX_CUDA(cudaMemcpyAsync(hc, c, 2 * sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        VX_CUDA(cudaStreamSynchronize(st));
        if (g_prof.on) {
            prof_elems(KC_SCATTER, hc[0].scat_elems);
            prof_elems(KC_FINISH, hc[0].fin_elems);
            prof_elems(KC_LOCAL, hc[0].loc_elems);
            prof_collect();
        }
        if (hc[0].err) return fail(VX_ECAPACITY, "sort work-queue capacity exceeded");
        nseg = hc[1].nseg;
        if (nseg == 0 && hc[1].fin_ctr == 0) return VX_OK;
    }
    return fail(VX_ECAPACITY, "sort exceeded the maximum level count");
}

// -------------------------------------------------------------- partition
// Tile shape of the pivot partition.  Measured on B200 (c3, 2^28 f64,
// kernel time).  With the decoupled look-back (VX_PART_LOOKBACK): 256x8
// 2.36 ms, 256x16 1.45, 512x16 1.30, 1024x16 1.19 -- larger tiles win, the
// look-back latency is exposed once per tile.  With run cursors (default):
// 1024x16 0.98, 512x16 0.77, 256x16 0.69, 128x16 0.67 ms (97 % of HBM
// peak), 128x32 0.70, 256x8 0.76 -- small tiles keep many CTAs per SM, so
// loads of one tile overlap the staging and stores of another.  The three
// cursors sit on separate L2 lines (on one line 128x16 ran 1.50 ms: the
// same-line atomics serialise).  Staging must fit in shared memory, so
// 16-byte pairs use half the tile.
template <typename K, typename V>
struct PartCfg {
    static constexpr int BYTES = sizeof(K) + (HasVal<V>::value ? sizeof(V) : 0);
#ifndef VX_PART_NT
#define VX_PART_NT 128
#endif
#ifndef VX_PART_IPT
#define VX_PART_IPT 16
#endif
    static constexpr int NT = VX_PART_NT;
    static constexpr int IPT = BYTES <= 8 ? VX_PART_IPT : VX_PART_IPT / 2;
};
constexpr uint64_t kPartMinTile = (uint64_t)VX_PART_NT * (VX_PART_IPT / 2);

template <typename K, typename V>
int run_partition(const K* kin, const V* vin, K* kout, V* vout, uint64_t n, K pivot, int64_t* d_split, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
    constexpr int NT = PartCfg<K, V>::NT, IPT = PartCfg<K, V>::IPT, T = NT * IPT;
    constexpr bool KV = HasVal<V>::value;
    if (n == 0) {
        VX_CUDA(cudaMemsetAsync(d_split, 0, sizeof(int64_t), st));
        return VX_OK;
    }
    const uint64_t ntiles = (n + T - 1) / T;
    const size_t need = align_up(ntiles * 8) + 512;
    if (!ws || ws_bytes < need) return fail(VX_EWORKSPACE, "partition workspace too small");
    auto* state = static_cast<unsigned long long*>(ws);
    auto* counter = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + align_up(ntiles * 8));
#ifdef VX_PART_LOOKBACK
    VX_CUDA(cudaMemsetAsync(ws, 0, need, st));
#else
    VX_CUDA(cudaMemsetAsync(counter, 0, 512, st));  // run cursors
#endif
    const size_t smem = (size_t)T * (sizeof(K) + (KV ? sizeof(V) : 0));
    const bool vec = ((reinterpret_cast<uintptr_t>(kin) | reinterpret_cast<uintptr_t>(vin)) & 15) == 0;
    auto* ds = reinterpret_cast<unsigned long long*>(d_split);
    Launch lch(KC_PARTITION, st);
    if (g_prof.on) prof_elems(KC_PARTITION, n);
    if (vec) {
        static int o1 = prepare(partition2_kernel<K, V, NT, IPT, true>, NT, smem);
        (void)o1;
        partition2_kernel<K, V, NT, IPT, true><<<(unsigned)ntiles, NT, smem, st>>>(kin, vin, kout, vout, n, pivot,
                                                                                 state, counter, ds);
    } else {
        static int o2 = prepare(partition2_kernel<K, V, NT, IPT, false>, NT, smem);
        (void)o2;
        partition2_kernel<K, V, NT, IPT, false><<<(unsigned)ntiles, NT, smem, st>>>(kin, vin, kout, vout, n, pivot,
                                                                                  state, counter, ds);
    }
    VX_LAUNCHED();
    return VX_OK;
}

// -------------------------------------------------------------- generators
template <typename K>
__global__ void gen_kernel(K* out, uint64_t n, int dist, uint64_t seed, uint64_t gofs, uint64_t gn) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = gofs + i;
        const uint64_t h = mix64(seed * 0xD1B54A32D192ED03ULL + g);
        if constexpr (sizeof(K) == 4) {
            int32_t v;
            switch (dist) {
                case 0: v = (int32_t)(uint32_t)(h >> 32); break;
                case 1: v = (int32_t)(uint32_t)(g * (0x100000000ULL / (gn ? gn : 1)) - 0x80000000ULL); break;
                case 2: v = (int32_t)(uint32_t)(0x7fffffffULL - g * (0x100000000ULL / (gn ? gn : 1))); break;
                case 3: v = (int32_t)(h >> 60); break;
                case 5: v = (int32_t)(h >> 33); break;
                default: v = (int32_t)(uint32_t)g; break;
            }
            out[i] = (K)v;
        } else {
            double v;
            switch (dist) {
                case 0: v = -1e6 + 2e6 * ((double)(h >> 11) * 0x1.0p-53); break;
                case 1: v = (double)g - 1073741824.0; break;
                case 2: v = 1073741823.0 - (double)g; break;
                case 3: v = (double)(h >> 60); break;
                case 4: {
                    const uint64_t h2 = mix64(h ^ 0xA0761D6478BD642FULL);
                    const double u1 = ((double)(h >> 11) + 1.0) * 0x1.0p-53;
                    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
                    v = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
                    if (v == 0.0) v = 0.0;  // never -0.0
                    break;
                }
                default: v = (double)g; break;
            }
            out[i] = (K)v;
        }
    }
}

// -------------------------------------------------------------- host arena
struct HostArena {
    std::mutex mu;
    void* p = nullptr;
    size_t cap = 0;
    cudaStream_t st = nullptr;
    int ensure(size_t bytes) {
        if (!st) VX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (bytes > cap) {
            if (p) VX_CUDA(cudaFree(p));
            p = nullptr;
            cap = 0;
            VX_CUDA(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return VX_OK;
    }
};
HostArena g_arena;

int check_dtype(int dtype) {
    if (dtype != VX_I32 && dtype != VX_F64) return fail(VX_ETYPE, "unsupported element dtype; use int32 or float64");
    return VX_OK;
}
inline size_t esize(int dtype) { return dtype == VX_I32 ? 4 : 8; }

int check_lane(int dtype, int64_t lane) {
    const int64_t want = dtype == VX_I32 ? 16 : 8;  // lanes.py:60-61
    if (lane != want) return fail(VX_EINVAL, "lane count does not match the element kind");
    return VX_OK;
}

int host_sort(int dtype, void* keys, void* vals, int64_t n, int64_t sort_bound, int strategy, int opt_a,
              int opt_b, uint64_t seed) {
    if (n < 2) return VX_OK;
    const size_t es = esize(dtype);
    const size_t data = align_up(n * es) * (vals ? 2 : 1);
    const size_t wsb = vx_sort_workspace_bytes(dtype, vals != nullptr, n);
    std::lock_guard<std::mutex> lk(g_arena.mu);
    int rc = g_arena.ensure(data + wsb);
    if (rc) return rc;
    char* d = static_cast<char*>(g_arena.p);
    void* dk = d;
    void* dv = vals ? d + align_up(n * es) : nullptr;
    cudaStream_t st = g_arena.st;
    VX_CUDA(cudaMemcpyAsync(dk, keys, n * es, cudaMemcpyHostToDevice, st));
    if (vals) VX_CUDA(cudaMemcpyAsync(dv, vals, n * es, cudaMemcpyHostToDevice, st));
    vx_sort_config cfg{sort_bound, strategy, opt_a, opt_b, 0, seed};
    rc = vx_sort(dtype, dk, dv, n, &cfg, d + data, wsb, (vx_stream_t)st);
    if (rc) return rc;
    VX_CUDA(cudaMemcpyAsync(keys, dk, n * es, cudaMemcpyDeviceToHost, st));
    if (vals) VX_CUDA(cudaMemcpyAsync(vals, dv, n * es, cudaMemcpyDeviceToHost, st));
    VX_CUDA(cudaStreamSynchronize(st));
    return VX_OK;
}

int64_t host_partition(int dtype, void* keys, void* vals, int64_t lo, int64_t hi, const void* pivot) {
    if (hi < lo || lo < 0) return fail(VX_EINVAL, "bad range");
    const int64_t n = hi - lo;
    if (n == 0) return lo;
    const size_t es = esize(dtype);
    char* hk = static_cast<char*>(keys) + lo * es;
    char* hv = vals ? static_cast<char*>(vals) + lo * es : nullptr;
    const size_t a = align_up(n * es);
    const size_t nbuf = vals ? 4 : 2;
    const size_t wsb = vx_partition_workspace_bytes(dtype, n);
    std::lock_guard<std::mutex> lk(g_arena.mu);
    int rc = g_arena.ensure(nbuf * a + 256 + wsb);
    if (rc) return rc;
    char* d = static_cast<char*>(g_arena.p);
    void* ik = d;
    void* ok = d + a;
    void* iv = vals ? d + 2 * a : nullptr;
    void* ov = vals ? d + 3 * a : nullptr;
    int64_t* dsplit = reinterpret_cast<int64_t*>(d + nbuf * a);
    cudaStream_t st = g_arena.st;
    VX_CUDA(cudaMemcpyAsync(ik, hk, n * es, cudaMemcpyHostToDevice, st));
    if (vals) VX_CUDA(cudaMemcpyAsync(iv, hv, n * es, cudaMemcpyHostToDevice, st));
    rc = vx_partition(dtype, ik, iv, ok, ov, n, pivot, dsplit, d + nbuf * a + 256, wsb, (vx_stream_t)st);
    if (rc) return rc;
    int64_t split = 0;
    VX_CUDA(cudaMemcpyAsync(hk, ok, n * es, cudaMemcpyDeviceToHost, st));
    if (vals) VX_CUDA(cudaMemcpyAsync(hv, ov, n * es, cudaMemcpyDeviceToHost, st));
    VX_CUDA(cudaMemcpyAsync(&split, dsplit, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    VX_CUDA(cudaStreamSynchronize(st));
    return lo + split;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* vx_last_error(void) { return g_err.c_str(); }
int vx_version(void) { return 1; }

size_t vx_sort_workspace_bytes(int dtype, int has_values, int64_t n) {
    if (n < 0) return 0;
    const uint64_t un = (uint64_t)n;
    if (dtype == VX_I32) return has_values ? SortLayout<int32_t, uint32_t>(un).total : SortLayout<int32_t, NoVal>(un).total;
    if (dtype == VX_F64) return has_values ? SortLayout<double, uint64_t>(un).total : SortLayout<double, NoVal>(un).total;
    return 0;
}

int vx_sort(int dtype, void* keys, void* values, int64_t n, const vx_sort_config* cfg, void* ws, size_t ws_bytes,
            vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 0 || (n > 0 && !keys)) return fail(VX_EINVAL, "bad array");
    return vx_sort_into(dtype, keys, values, keys, values, n, cfg, ws, ws_bytes, stream);
}

int vx_sort_into(int dtype, const void* in_keys, const void* in_values, void* out_keys, void* out_values, int64_t n,
                 const vx_sort_config* cfg, void* ws, size_t ws_bytes, vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 0 || (n > 0 && (!in_keys || !out_keys))) return fail(VX_EINVAL, "bad array");
    if ((in_values == nullptr) != (out_values == nullptr)) return fail(VX_EINVAL, "values in/out mismatch");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == VX_I32) {
        if (in_values)
            return run_sort<int32_t, uint32_t>((const int32_t*)in_keys, (const uint32_t*)in_values, (int32_t*)out_keys,
                                               (uint32_t*)out_values, n, cfg, ws, ws_bytes, st);
        return run_sort<int32_t, NoVal>((const int32_t*)in_keys, nullptr, (int32_t*)out_keys, nullptr, n, cfg, ws,
                                        ws_bytes, st);
    }
    if (in_values)
        return run_sort<double, uint64_t>((const double*)in_keys, (const uint64_t*)in_values, (double*)out_keys,
                                          (uint64_t*)out_values, n, cfg, ws, ws_bytes, st);
    return run_sort<double, NoVal>((const double*)in_keys, nullptr, (double*)out_keys, nullptr, n, cfg, ws, ws_bytes,
                                   st);
}

int vx_profile_enable(int on) {
    prof_collect();
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    return VX_OK;
}

int vx_profile_reset(void) {
    prof_collect();
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (int i = 0; i < KC_N; ++i) {
        g_prof.launches[i] = 0;
        g_prof.ms[i] = 0.0;
        g_prof.elems[i] = 0;
    }
    return VX_OK;
}

int vx_profile_read(int64_t* launches, double* ms, uint64_t* elems, int nclass) {
    prof_collect();
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (int i = 0; i < nclass && i < KC_N; ++i) {
        if (launches) launches[i] = g_prof.launches[i];
        if (ms) ms[i] = g_prof.ms[i];
        if (elems) elems[i] = g_prof.elems[i];
    }
    return KC_N;
}

size_t vx_partition_workspace_bytes(int dtype, int64_t n) {
    (void)dtype;
    const uint64_t T = kPartMinTile;
    return align_up(((uint64_t)n + T - 1) / T * 8) + 512;
}

int vx_partition(int dtype, const void* in_keys, const void* in_values, void* out_keys, void* out_values, int64_t n,
                 const void* pivot, int64_t* d_split, void* ws, size_t ws_bytes, vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 0 || !pivot || !d_split || (n > 0 && (!in_keys || !out_keys))) return fail(VX_EINVAL, "bad argument");
    if ((in_values == nullptr) != (out_values == nullptr)) return fail(VX_EINVAL, "values in/out mismatch");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == VX_I32) {
        const int32_t p = *static_cast<const int32_t*>(pivot);
        if (in_values)
            return run_partition<int32_t, uint32_t>((const int32_t*)in_keys, (const uint32_t*)in_values,
                                                    (int32_t*)out_keys, (uint32_t*)out_values, n, p, d_split, ws,
                                                    ws_bytes, st);
        return run_partition<int32_t, NoVal>((const int32_t*)in_keys, nullptr, (int32_t*)out_keys, nullptr, n, p,
                                             d_split, ws, ws_bytes, st);
    }
    const double p = *static_cast<const double*>(pivot);
    if (in_values)
        return run_partition<double, uint64_t>((const double*)in_keys, (const uint64_t*)in_values, (double*)out_keys,
                                               (uint64_t*)out_values, n, p, d_split, ws, ws_bytes, st);
    return run_partition<double, NoVal>((const double*)in_keys, nullptr, (double*)out_keys, nullptr, n, p, d_split,
                                        ws, ws_bytes, st);
}

int vx_sort_segments(int dtype, void* keys, void* values, const int64_t* d_offsets, int64_t nseg, void* ws,
                     size_t ws_bytes, vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (nseg < 0 || (nseg > 0 && (!keys || !d_offsets))) return fail(VX_EINVAL, "bad argument");
    if (!ws || ws_bytes < 4) return fail(VX_EWORKSPACE, "segments workspace must hold 4 bytes");
    cudaStream_t st = (cudaStream_t)stream;
    VX_CUDA(cudaMemsetAsync(ws, 0, 4, st));
    if (nseg == 0) return VX_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((nseg + 7) / 8, (int64_t)num_sms() * 16);
    auto* err = static_cast<unsigned*>(ws);
    const auto* offs = reinterpret_cast<const long long*>(d_offsets);
    Launch lch(KC_SEGSORT, st);
    if (dtype == VX_I32) {
        if (values) segsort_kernel<int32_t, uint32_t><<<grid, 256, 0, st>>>((int32_t*)keys, (uint32_t*)values, offs, nseg, err);
        else segsort_kernel<int32_t, NoVal><<<grid, 256, 0, st>>>((int32_t*)keys, nullptr, offs, nseg, err);
    } else {
        if (values) segsort_kernel<double, uint64_t><<<grid, 256, 0, st>>>((double*)keys, (uint64_t*)values, offs, nseg, err);
        else segsort_kernel<double, NoVal><<<grid, 256, 0, st>>>((double*)keys, nullptr, offs, nseg, err);
    }
    VX_LAUNCHED();
    return VX_OK;
}

int vx_segments_status(void* ws, vx_stream_t stream) {
    unsigned e = 0;
    VX_CUDA(cudaMemcpyAsync(&e, ws, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    VX_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (e & kErrTooLong) return fail(VX_ETOOLONG, "region exceeds small-sort capacity (256)");
    return VX_OK;
}

size_t vx_bucket_partition_workspace_bytes(int dtype, int nsplit) {
    (void)dtype;
    return align_up((size_t)(nsplit + 1) * 8);
}

int vx_bucket_partition(int dtype, const void* in_keys, void* out_keys, int64_t n, uint64_t global_offset,
                        const void* d_split_keys, const uint64_t* d_split_idx, int nsplit,
                        unsigned long long* d_counts, void* ws, size_t ws_bytes, vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (nsplit < 0 || nsplit > kMaxSplit || n < 0 || !d_counts) return fail(VX_EINVAL, "bad argument");
    if (!ws || ws_bytes < vx_bucket_partition_workspace_bytes(dtype, nsplit)) return fail(VX_EWORKSPACE, "workspace");
    cudaStream_t st = (cudaStream_t)stream;
    auto* cursor = static_cast<unsigned long long*>(ws);
    VX_CUDA(cudaMemsetAsync(d_counts, 0, (nsplit + 1) * 8, st));
    if (n == 0) return VX_OK;
    const int sms = num_sms();
    Launch lch(KC_BUCKET, st, 3);
    if (g_prof.on) prof_elems(KC_BUCKET, n);
    if (dtype == VX_I32) {
        using K = int32_t;
        static int occ = prepare(bp_scatter_kernel<K, NoVal>, kQsNT, sizeof(ScatterSmem<K, NoVal>));
        bp_hist_kernel<K><<<sms * 8, kQsNT, 0, st>>>((const K*)in_keys, n, global_offset, (const K*)d_split_keys,
                                                    d_split_idx, nsplit, d_counts);
        bp_scan_kernel<<<1, 32, 0, st>>>(d_counts, nsplit + 1, cursor);
        bp_scatter_kernel<K, NoVal><<<sms * occ, kQsNT, sizeof(ScatterSmem<K, NoVal>), st>>>(
            (const K*)in_keys, nullptr, (K*)out_keys, nullptr, n, global_offset, (const K*)d_split_keys, d_split_idx,
            nsplit, cursor);
    } else {
        using K = double;
        static int occ = prepare(bp_scatter_kernel<K, NoVal>, kQsNT, sizeof(ScatterSmem<K, NoVal>));
        bp_hist_kernel<K><<<sms * 8, kQsNT, 0, st>>>((const K*)in_keys, n, global_offset, (const K*)d_split_keys,
                                                    d_split_idx, nsplit, d_counts);
        bp_scan_kernel<<<1, 32, 0, st>>>(d_counts, nsplit + 1, cursor);
        bp_scatter_kernel<K, NoVal><<<sms * occ, kQsNT, sizeof(ScatterSmem<K, NoVal>), st>>>(
            (const K*)in_keys, nullptr, (K*)out_keys, nullptr, n, global_offset, (const K*)d_split_keys, d_split_idx,
            nsplit, cursor);
    }
    VX_LAUNCHED();
    return VX_OK;
}

int vx_select_splitters(int dtype, const void* d_sample_keys, const uint64_t* d_sample_idx, int64_t count,
                        int nparts, void* d_out_keys, uint64_t* d_out_idx, vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (count < 1 || count > 8192 || nparts < 1 || nparts > kMaxSplit + 1) return fail(VX_EINVAL, "bad sample count");
    if (nparts == 1) return VX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t P = next_pow2_u32((uint32_t)count);
    if (dtype == VX_I32) {
        const size_t smem = P * (4 + 8);
        prepare(select_splitters_kernel<int32_t>, 1024, smem);
        select_splitters_kernel<int32_t><<<1, 1024, smem, st>>>((const int32_t*)d_sample_keys, d_sample_idx,
                                                                (unsigned)count, nparts, (int32_t*)d_out_keys,
                                                                d_out_idx);
    } else {
        const size_t smem = P * (8 + 8);
        prepare(select_splitters_kernel<double>, 1024, smem);
        select_splitters_kernel<double><<<1, 1024, smem, st>>>((const double*)d_sample_keys, d_sample_idx,
                                                               (unsigned)count, nparts, (double*)d_out_keys, d_out_idx);
    }
    VX_LAUNCHED();
    return VX_OK;
}

int vx_generate(int dtype, int dist, void* out, int64_t n, uint64_t seed, uint64_t global_offset, int64_t global_n,
                vx_stream_t stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 0 || dist < 0 || dist > 6) return fail(VX_EINVAL, "bad generator argument");
    if (n == 0) return VX_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 32);
    if (dtype == VX_I32)
        gen_kernel<int32_t><<<grid, 256, 0, (cudaStream_t)stream>>>((int32_t*)out, n, dist, seed, global_offset,
                                                                    (uint64_t)global_n);
    else
        gen_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>((double*)out, n, dist, seed, global_offset,
                                                                   (uint64_t)global_n);
    VX_LAUNCHED();
    return VX_OK;
}

// ------------------------------------------------------------ host drop-in
int vx_host_quicksort(int dtype, void* arr, int64_t n, int64_t lane, int64_t sort_bound, int strategy, int opt_a,
                      int opt_b, uint64_t seed) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_lane(dtype, lane)) return rc;
    if (strategy < 0 || strategy > 2) return fail(VX_EINVAL, "unknown pivot strategy");
    return host_sort(dtype, arr, nullptr, n, sort_bound, strategy, opt_a, opt_b, seed);
}

int vx_host_kv_quicksort(int dtype, void* keys, void* vals, int64_t n, int64_t lane, int64_t sort_bound,
                         int strategy, int opt_a, int opt_b, uint64_t seed) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_lane(dtype, lane)) return rc;
    if (!vals) return fail(VX_EINVAL, "values required");
    return host_sort(dtype, keys, vals, n, sort_bound, strategy, opt_a, opt_b, seed);
}

int64_t vx_host_partition(int dtype, void* arr, int64_t lo, int64_t hi, const void* pivot, int64_t lane, int opt_a,
                          int opt_b) {
    (void)opt_a;
    (void)opt_b;
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_lane(dtype, lane)) return rc;
    return host_partition(dtype, arr, nullptr, lo, hi, pivot);
}

int64_t vx_host_kv_partition(int dtype, void* keys, void* vals, int64_t lo, int64_t hi, const void* pivot,
                             int64_t lane, int opt_a, int opt_b) {
    (void)opt_a;
    (void)opt_b;
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_lane(dtype, lane)) return rc;
    return host_partition(dtype, keys, vals, lo, hi, pivot);
}

int64_t vx_host_scalar_partition(int dtype, void* arr, int64_t lo, int64_t hi, const void* pivot) {
    if (int rc = check_dtype(dtype)) return rc;
    return host_partition(dtype, arr, nullptr, lo, hi, pivot);
}

int64_t vx_host_kv_scalar_partition(int dtype, void* keys, void* vals, int64_t lo, int64_t hi, const void* pivot) {
    if (int rc = check_dtype(dtype)) return rc;
    return host_partition(dtype, keys, vals, lo, hi, pivot);
}

int vx_host_smallsort_region(int dtype, void* arr, int64_t lo, int64_t length) {
    if (int rc = check_dtype(dtype)) return rc;
    if (length < 2) return VX_OK;
    const size_t es = esize(dtype);
    return host_sort(dtype, static_cast<char*>(arr) + lo * es, nullptr, length, 0, 0, 0, 0, 0);
}

int vx_host_kv_smallsort_region(int dtype, void* keys, void* vals, int64_t lo, int64_t length) {
    if (int rc = check_dtype(dtype)) return rc;
    if (length < 2) return VX_OK;
    const size_t es = esize(dtype);
    return host_sort(dtype, static_cast<char*>(keys) + lo * es, static_cast<char*>(vals) + lo * es, length, 0, 0, 0,
                     0, 0);
}

int vx_host_release(void) {
    std::lock_guard<std::mutex> lk(g_arena.mu);
    if (g_arena.p) VX_CUDA(cudaFree(g_arena.p));
    g_arena.p = nullptr;
    g_arena.cap = 0;
    return VX_OK;
}

}  // extern "C"
