// C ABI of libqsb200.so: state lifetime, the fusion planner, observables and
// the global-qubit exchange (declarations and reference citations in
// include/qsb200.h).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"

#include <atomic>

using namespace qsb;

// Every host-blocking CUDA call of the library goes through these; the count
// is exported (qs_host_sync_count) so tests can show that the global-qubit
// path never blocks the host between gates (its exchange kernels are ordered
// by CUDA events, not host syncs).
namespace {
std::atomic<uint64_t> g_host_syncs{0};
inline cudaError_t host_sync_stream(cudaStream_t s) {
    g_host_syncs.fetch_add(1, std::memory_order_relaxed);
    return cudaStreamSynchronize(s);
}
inline cudaError_t host_sync_event(cudaEvent_t e) {
    g_host_syncs.fetch_add(1, std::memory_order_relaxed);
    return cudaEventSynchronize(e);
}
inline cudaError_t host_sync_device() {
    g_host_syncs.fetch_add(1, std::memory_order_relaxed);
    return cudaDeviceSynchronize();
}
}  // namespace

namespace qsb {
size_t tile_smem_bytes();
int prof_read(unsigned long long* out);
}

// ---------------------------------------------------------------------------
// errors
namespace {
thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) {                                                          \
            (void)cudaGetLastError(); /* a non-sticky error must not resurface later */   \
            return fail(_e == cudaErrorMemoryAllocation ? QS_ERR_NOMEM : QS_ERR_CUDA,    \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
        }                                                                                 \
    } while (0)

#define CHECK_LAUNCH()                                                                    \
    do {                                                                                  \
        cudaError_t _e = cudaGetLastError();                                              \
        if (_e != cudaSuccess)                                                            \
            return fail(QS_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                              \
    } while (0)

// ---------------------------------------------------------------------------
// NCCL, loaded lazily so the library has no link-time dependency on a
// particular libnccl (torch ships its own).
typedef int ncclResult_t_;
typedef void* ncclComm_t_;
struct NcclId {
    char internal[128];
};
enum { kNcclFloat64 = 8 };  // ncclDataType_t: ncclFloat64 == ncclDouble == 8

struct NcclApi {
    bool loaded = false;
    void* handle = nullptr;
    ncclResult_t_ (*GetUniqueId)(NcclId*) = nullptr;
    ncclResult_t_ (*CommInitRank)(ncclComm_t_*, int, NcclId, int) = nullptr;
    ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
    ncclResult_t_ (*Send)(const void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
    ncclResult_t_ (*Recv)(void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
    ncclResult_t_ (*GroupStart)() = nullptr;
    ncclResult_t_ (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t_) = nullptr;
};
NcclApi g_nccl;

std::mutex g_nccl_mutex;

int nccl_load() {
    std::lock_guard<std::mutex> lock(g_nccl_mutex);  // ranks may be threads
    if (g_nccl.loaded) return QS_OK;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        g_nccl.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.handle) break;
    }
    if (!g_nccl.handle) return fail(QS_ERR_COMM, "cannot dlopen libnccl.so.2: %s", dlerror());
#define NCCL_SYM(field, name)                                                          \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(g_nccl.handle, name)); \
    if (!g_nccl.field) return fail(QS_ERR_COMM, "libnccl lacks %s", name);
    NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    NCCL_SYM(CommInitRank, "ncclCommInitRank");
    NCCL_SYM(CommDestroy, "ncclCommDestroy");
    NCCL_SYM(Send, "ncclSend");
    NCCL_SYM(Recv, "ncclRecv");
    NCCL_SYM(GroupStart, "ncclGroupStart");
    NCCL_SYM(GroupEnd, "ncclGroupEnd");
    NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef NCCL_SYM
    g_nccl.loaded = true;
    return QS_OK;
}

#define NCCL_TRY(expr)                                                                     \
    do {                                                                                   \
        ncclResult_t_ _r = (expr);                                                         \
        if (_r != 0)                                                                       \
            return fail(QS_ERR_COMM, "%s: %s", #expr, g_nccl.GetErrorString(_r));          \
    } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// state
struct LaunchRec {
    int32_t kind;
    cudaEvent_t start, stop;
};

struct qs_state {
    int n = 0, m = 0, rank = 0, num_states = 1, device = 0;
    uint64_t amps_per_state = 0;
    double2* psi = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t comm_stream = nullptr;
    // device scratch
    double* d_mats = nullptr;
    size_t mats_cap = 0;  // doubles
    TilePass* d_pass = nullptr;
    size_t pass_cap = 0;
    double* d_scratch = nullptr;
    size_t scratch_cap = 0;
    double* d_u = nullptr;  // 8 doubles for exchange gates
    double* h_out = nullptr;  // pinned observable results
    size_t h_out_cap = 0;
    // NCCL exchange staging
    ncclComm_t_ comm = nullptr;
    double2* d_stage[2] = {nullptr, nullptr};
    size_t stage_cap = 0;  // amplitudes per buffer
    // accounting (TransportCounters analogue)
    uint64_t messages = 0, amplitudes = 0;
    int32_t last_passes = 0;
    // cross-rank ordering of exchange kernels (qs_sync_event*): interprocess
    // events recorded before / after an exchange; peer events opened here
    cudaEvent_t sync_ev[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> opened_ev;
    // NCCL exchange pipeline events, created once
    cudaEvent_t nccl_ev[6] = {};
    // timing
    cudaEvent_t ev[8] = {};
    bool launch_log = false;
    std::vector<LaunchRec> recs;
};

namespace {

int ensure_device(qs_state* st) {
    CUDA_TRY(cudaSetDevice(st->device));
    return QS_OK;
}

template <typename T>
int grow(T** p, size_t* cap, size_t need) {
    if (*cap >= need) return QS_OK;
    if (*p) {
        host_sync_device();  // queued kernels may still read the old buffer
        cudaError_t e = cudaFree(*p);
        if (e != cudaSuccess) return fail(QS_ERR_CUDA, "cudaFree: %s", cudaGetErrorString(e));
    }
    size_t n = std::max(need, *cap * 2);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // clear the (non-sticky) allocation error
        *p = nullptr;
        *cap = 0;
        return fail(QS_ERR_NOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
    }
    *cap = n;
    return QS_OK;
}

int build_cut_terms(const int32_t* edges, int32_t num_edges, int n, CutTerms* ct) {
    memset(ct, 0, sizeof(*ct));
    if (num_edges < 0) return fail(QS_ERR_VALUE, "negative edge count");
    if (num_edges > 0 && !edges) return fail(QS_ERR_VALUE, "edges is NULL");
    for (int e = 0; e < num_edges; ++e) {
        int u = edges[2 * e], v = edges[2 * e + 1];
        if (u == v) return fail(QS_ERR_VALUE, "self-loop at vertex %d", u);
        if (u < 0 || v < 0 || u >= n || v >= n || u > 63 || v > 63)
            return fail(QS_ERR_VALUE, "edge (%d, %d) endpoint out of range for %d qubits", u, v, n);
        int lo = std::min(u, v), d = std::abs(u - v);
        int k = 0;
        while (k < ct->count && ct->shift[k] != d) ++k;
        if (k == ct->count) {
            if (ct->count == kMaxCutTerms) return fail(QS_ERR_VALUE, "too many edge distances");
            ct->shift[k] = d;
            ct->mask[k] = 0;
            ct->count++;
        }
        if (ct->mask[k] & (uint64_t(1) << lo))
            return fail(QS_ERR_VALUE, "duplicate edge (%d, %d)", u, v);
        ct->mask[k] |= uint64_t(1) << lo;
    }
    return QS_OK;
}

// launch bracketing for the optional per-launch timing log
struct LaunchScope {
    qs_state* st;
    LaunchRec rec{};
    bool cancelled = false;  // nothing was launched: no record
    LaunchScope(qs_state* s, int kind) : st(s) {
        if (!st->launch_log) return;
        rec.kind = kind;
        cudaEventCreate(&rec.start);
        cudaEventCreate(&rec.stop);
        cudaEventRecord(rec.start, st->stream);
    }
    ~LaunchScope() {
        if (!st->launch_log) return;
        if (cancelled) {
            cudaEventDestroy(rec.start);
            cudaEventDestroy(rec.stop);
            return;
        }
        cudaEventRecord(rec.stop, st->stream);
        st->recs.push_back(rec);
    }
};

enum { kLaunchGate1q = 1, kLaunchControlled = 2, kLaunchPhase = 3, kLaunchTile = 4,
       kLaunchExchange = 5, kLaunchReduce = 6, kLaunchFact = 7,
       kLaunchFactGen = 8 /* lean pass with a generated (constant) input: write-only */,
       kLaunchPerm = 9 /* CNOT-only pass of a factored program as one permutation (k_perm) */ };

bool is_diag_one(const double* e) {
    return e[0] == 1.0 && e[1] == 0.0 && e[2] == 0.0 && e[3] == 0.0 && e[4] == 0.0 && e[5] == 0.0;
}

// ---- the fusion planner ----------------------------------------------------
thread_local uint64_t g_zero_off = 0;  // factored program being launched: a 0.0 in mats
thread_local bool g_factored = false;  // the program being launched is a factored rewrite
struct PlannedPass {
    int first, count;  // range in the program
};

int launch_single(qs_state* st, const qs_gate& g, const CutTerms& ct, const double* mats_host) {
    const int ns = st->num_states;
    if (g.kind == QS_KIND_1Q) {
        LaunchScope ls(st, kLaunchGate1q);
        launch_gate1q(st->psi, st->m, ns, g.target, st->d_mats, g.offset, g.stride, st->stream);
    } else if (g.kind == QS_KIND_CTRL) {
        bool diag = true;
        for (int s = 0; s < ns && diag; ++s) diag = is_diag_one(mats_host + g.offset + s * g.stride);
        LaunchScope ls(st, kLaunchControlled);
        launch_controlled(st->psi, st->m, ns, g.control, g.target, st->d_mats, g.offset, g.stride,
                          diag, st->stream);
    } else {
        LaunchScope ls(st, kLaunchPhase);
        launch_cut_phase(st->psi, st->m, ns, uint64_t(st->rank) << st->m, ct, st->d_mats, g.offset,
                         g.stride, st->stream);
    }
    CHECK_LAUNCH();
    return QS_OK;
}



// Build the TilePass for program[first, first+count) and launch it.
int launch_tile(qs_state* st, const qs_gate* prog, int first, int count, const CutTerms& ct,
                const double* mats_host) {
    if (count > kMaxPassGates) return fail(QS_ERR_VALUE, "planner: pass too long");
    if (g_factored && st->num_states == 1) {
        // a pass of CNOTs only is a permutation of the index bits: one gather
        // per 2^13-amplitude box at copy speed, whatever the number of gates
        // (factored programs: the exact mode keeps numpy's signed zeros)
        static const double kX[8] = {0, 0, 1, 0, 1, 0, 0, 0};
        int cs[kMaxPassGates], ts[kMaxPassGates];
        bool all_x = true;
        for (int i = 0; i < count && all_x; ++i) {
            const qs_gate& g = prog[first + i];
            all_x = g.kind == QS_KIND_CTRL && g.stride == 0 &&
                    memcmp(mats_host + g.offset, kX, sizeof(kX)) == 0;
            cs[i] = g.control;
            ts[i] = g.target;
        }
        if (all_x) {
            if (g_const_in.on) {  // the permutation reads its input from HBM
                launch_fill(st->psi, g_const_in.total, g_const_in.v, st->stream);
                g_const_in.on = false;
            }
            LaunchScope ls(st, kLaunchPerm);
            if (launch_perm(st->psi, st->m, cs, ts, count, st->stream)) {
                CHECK_LAUNCH();
                return QS_OK;
            }
            ls.cancelled = true;
        }
    }
    // tile bits: the targets, plus qubits 0..2 for 128-byte rows, filled upward
    uint64_t need = kLowMask;
    for (int i = 0; i < count; ++i)
        if (kind_has_target(prog[first + i].kind)) need |= uint64_t(1) << prog[first + i].target;
    static thread_local bool no_absorb_fill = false;
    bool absorb_fill = false;
    if (g_absorb.count > 0 && !no_absorb_fill) {
        // spare tile bits go to the targets of the CNOT pass behind this one, so
        // that it can be folded into this pass (all of them or none); checked
        // below: a tile the lean TMA kernel cannot take falls back to the plain fill
        uint64_t want = need;
        for (int i = 0; i < g_absorb.count; ++i) want |= uint64_t(1) << g_absorb.targets[i];
        if (__builtin_popcountll(want) <= kTileLog2 && want != need) need = want, absorb_fill = true;
    }
    for (int b = 0; __builtin_popcountll(need) < kTileLog2 && b < st->m; ++b) need |= uint64_t(1) << b;
    static thread_local TilePass P;
    memset(&P, 0, sizeof(P));
    P.m = st->m;
    int k = 0;
    for (int b = 0; b < st->m; ++b)
        if (need & (uint64_t(1) << b)) P.tile_bits[k++] = b;
    P.low_run = 0;
    while (P.low_run < kTileLog2 && P.tile_bits[P.low_run] == P.low_run) ++P.low_run;
    P.tiles_per_state = uint64_t(1) << (st->m - kTileLog2);
    P.num_tiles = P.tiles_per_state * uint64_t(st->num_states);
    P.rank_offset = uint64_t(st->rank) << st->m;
    P.zero_off = g_zero_off;
    for (int k = 0; k < ct.count; ++k)
        for (int u = 0; u < 64; ++u)
            if ((ct.mask[k] >> u) & 1) {
                const int v = u + ct.shift[k];
                P.nbr[u] |= uint64_t(1) << v;
                P.nbr[v] |= uint64_t(1) << u;
            }
    auto pos_of = [&](int qubit) {
        for (int p = 0; p < kTileLog2; ++p)
            if (P.tile_bits[p] == qubit) return p;
        return -1;
    };
    // rounds: consecutive gates whose targets fit in kRegLog2 register positions
    std::vector<int> round_pos;
    std::vector<std::vector<int>> all_pos;
    int r = -1;
    auto close_round = [&]() {
        if (r < 0) return;
        // pad with the highest unused positions so the lanes keep the low positions
        uint32_t used = 0;
        for (int p : round_pos) used |= 1u << p;
        for (int p = kTileLog2 - 1; (int)round_pos.size() < kRegLog2 && p >= 0; --p)
            if (!(used & (1u << p))) round_pos.push_back(p), used |= 1u << p;
        Round& R = P.rounds[r];
        int nonround[kTileLog2 - kRegLog2], c = 0;
        for (int p = 0; p < kTileLog2; ++p)
            if (!(used & (1u << p))) nonround[c++] = p;
        // lanes 0..2 (a quarter warp) should differ in the swizzle's bank bit
        // (position p moves bank bit p mod 3): pull forward the first positions
        // of distinct classes, keeping ascending order otherwise (when 0,1,2 are
        // all lanes nothing moves, so direct stores stay 128-byte rows)
        {
            int picked[3], np = 0;
            unsigned cls = 0;
            for (int i = 0; i < c && np < 3; ++i)
                if (!(cls & (1u << (nonround[i] % 3)))) {
                    cls |= 1u << (nonround[i] % 3);
                    picked[np++] = i;
                }
            if (np == 3) {
                int reordered[kTileLog2 - kRegLog2], n2 = 0;
                for (int j = 0; j < 3; ++j) reordered[n2++] = nonround[picked[j]];
                for (int i = 0; i < c; ++i)
                    if (i != picked[0] && i != picked[1] && i != picked[2]) reordered[n2++] = nonround[i];
                for (int i = 0; i < c; ++i) nonround[i] = reordered[i];
            }
        }
        auto deposit = [](int v, const int* pos, int nbits) {
            int out = 0;
            for (int b = 0; b < nbits; ++b)
                if ((v >> b) & 1) out |= 1 << pos[b];
            return out;
        };
        for (int v = 0; v < (1 << kLaneLoBits); ++v) {
            R.dlo[v] = uint16_t(deposit(v, nonround, kLaneLoBits));
            R.slo[v] = uint16_t(swz(R.dlo[v]));
        }
        for (int v = 0; v < (1 << kLaneHiBits); ++v) {
            R.dhi[v] = uint16_t(deposit(v, nonround + kLaneLoBits, kLaneHiBits));
            R.shi[v] = uint16_t(swz(R.dhi[v]));
        }
        for (int v = 0; v < (1 << kRegLog2); ++v) {
            R.dk[v] = uint16_t(deposit(v, round_pos.data(), kRegLog2));
            R.sk[v] = uint16_t(swz(R.dk[v]));
        }
        all_pos.push_back(round_pos);
    };
    std::vector<int> gate_round(count);
    for (int i = 0; i < count; ++i) {
        const qs_gate& g = prog[first + i];
        int p = kind_has_target(g.kind) ? pos_of(g.target) : -1;
        bool fits = r >= 0;
        if (fits && p >= 0 &&
            std::find(round_pos.begin(), round_pos.end(), p) == round_pos.end() &&
            (int)round_pos.size() >= kRegLog2)
            fits = false;
        if (!fits) {
            close_round();
            ++r;
            if (r >= kMaxRounds) return fail(QS_ERR_VALUE, "planner: too many rounds");
            round_pos.clear();
            P.rounds[r].first_gate = int16_t(i);
            P.rounds[r].num_gates = 0;
        }
        if (p >= 0 && std::find(round_pos.begin(), round_pos.end(), p) == round_pos.end())
            round_pos.push_back(p);
        P.rounds[r].num_gates++;
        gate_round[i] = r;
    }
    close_round();
    P.num_rounds = r + 1;
    {
        // the last round can store straight from registers when its lanes cover
        // tile positions 0,1,2 (i.e. none of them is held in registers)
        bool low_free = true;
        for (int p : all_pos.back())
            if (p < 3) low_free = false;
        P.direct_store = (low_free && P.low_run >= 3 && kLowBits >= 3) ? 1 : 0;
    }
    int ndiag = 0;
    for (int i = 0; i < count; ++i) {
        const qs_gate& g = prog[first + i];
        TileGate& d = P.gates[i];
        d.kind = g.kind;
        d.offset = g.offset;
        d.stride = g.stride;
        d.variant = 0;
        d.ctype = 0;
        d.cval = 0;
        d.seq = 0;
        if (g.kind == QS_KIND_CUTPHASE) continue;
        if (g.kind == kKindDiagN) {
            d.cval = g.reserved;  // byte-table count
            // register part of the diagonal for this round: R[k] = prod_j z_{q_j}^{k_j}
            const int slot = ndiag++;
            if (slot >= kMaxPassDiags) return fail(QS_ERR_VALUE, "planner: too many diagonals");
            d.pad[0] = slot;
            const double* z = mats_host + g.offset + 512 * uint64_t(g.reserved);
            const std::vector<int>& rp = all_pos[gate_round[i]];
            double2* R = P.diag_r[slot];
            R[0] = make_double2(1.0, 0.0);
            for (int k = 1; k < (1 << kRegLog2); ++k) {
                const int h = 31 - __builtin_clz(k);
                const int q = P.tile_bits[rp[h]];
                const double2 x = R[k ^ (1 << h)];
                const double zr = z[2 * q], zi = z[2 * q + 1];
                R[k] = make_double2(x.x * zr - x.y * zi, x.x * zi + x.y * zr);
            }
            continue;
        }
        // per-state shears: the first state's row (the pre-diagonal is shared
        // by construction; t is read per state)
        if (g.stride == 0 || g.kind == kKindShear)
            memcpy(&d.u[0], mats_host + g.offset, 8 * sizeof(double));
        if (g.kind == kKindScalar) continue;
        if (g.kind == kKindShear) d.pad[1] = g.reserved;  // 1: per-state pre-diagonals
        const std::vector<int>& rp = all_pos[gate_round[i]];
        int p = pos_of(g.target), j = 0;
        for (int jj = 0; jj < kRegLog2; ++jj)
            if (rp[jj] == p) j = jj;
        d.variant = j;
        if (g.kind == QS_KIND_CTRL) {
            int pc = pos_of(g.control);
            if (pc < 0) {
                d.ctype = 3;
                d.cval = g.control;
            } else {
                int jc = -1;
                for (int jj = 0; jj < kRegLog2; ++jj)
                    if (rp[jj] == pc) jc = jj;
                d.ctype = jc >= 0 ? 1 : 2;
                d.cval = jc >= 0 ? jc : pc;
                if (jc >= 0) d.variant = kRegLog2 + kRegLog2 * jc + j;
            }
        }
    }
    // mark runs of uncontrolled gates (or of shears) on register bits 0,1,2,..
    // (in order, same round)
    for (int i = 0; i < count;) {
        int n = 0;
        const int kind = P.gates[i].kind;
        while (i + n < count && n < kRegLog2 && (kind == QS_KIND_1Q || kind == kKindShear) &&
               P.gates[i + n].kind == kind && P.gates[i + n].variant == n &&
               gate_round[i + n] == gate_round[i])
            ++n;
        if (n >= 1) {
            P.gates[i].seq = n;
            i += n;
        } else {
            ++i;
        }
    }
    if (absorb_fill && !absorb_tile_feasible(st->psi, P)) {
        no_absorb_fill = true;
        const int rc = launch_tile(st, prog, first, count, ct, mats_host);
        no_absorb_fill = false;
        return rc;
    }
    static const bool debug_plan = getenv("QSB_DEBUG_PLAN") != nullptr;
    if (debug_plan) {  // one line per pass: rounds as [gate kind:target ...]
        fprintf(stderr, "pass tile=");
        for (int b = 0; b < kTileLog2; ++b) fprintf(stderr, "%d%s", P.tile_bits[b], b + 1 < kTileLog2 ? "," : "");
        for (int rr = 0; rr < P.num_rounds; ++rr) {
            fprintf(stderr, " [");
            for (int g = P.rounds[rr].first_gate; g < P.rounds[rr].first_gate + P.rounds[rr].num_gates; ++g) {
                fprintf(stderr, "%s%d:%d", g > P.rounds[rr].first_gate ? " " : "", P.gates[g].kind,
                        prog[first + g].target);
                if (P.gates[g].kind == QS_KIND_CTRL) fprintf(stderr, "/c%d", P.gates[g].ctype);
            }
            fprintf(stderr, "]");
        }
        fprintf(stderr, "\n");
    }
    if (!tile_pass_in_params()) {  // QSB_PASS_SMEM builds read the pass from a device copy
        if (int rc = grow(&st->d_pass, &st->pass_cap, 1)) return rc;
        CUDA_TRY(cudaMemcpyAsync(st->d_pass, &P, sizeof(P), cudaMemcpyHostToDevice, st->stream));
    }
    {
        LaunchScope ls(st, kLaunchTile);
        const int lean = launch_tile_pass(st->psi, P, st->d_pass, st->d_mats, ct, st->stream);
        if (lean) ls.rec.kind = lean == 2 ? kLaunchFactGen : kLaunchFact;
    }
    CHECK_LAUNCH();
    return QS_OK;
}

// Greedy pass formation (the native fusion planner).  A pass grows while
//  * the union of its target qubits plus qubits 0..2 (128-byte rows) fits the
//    2^kTileLog2-amplitude tile, and
//  * its register rounds (consecutive gates touching <= kRegLog2 distinct
//    targets) stay within kMaxRounds.
// Phase gates need no tile bit.  Single-gate passes use the streaming kernels.
struct PassPlan {
    int first, count;
};

std::vector<PassPlan> plan_passes(const qs_gate* gates, int count, int m, bool fuse,
                                  bool lean_first = false, const double* mats = nullptr) {
    std::vector<PassPlan> out;
    const bool tile_ok = fuse && m >= kTileLog2;
    int i = 0;
    while (i < count) {
        int j = i + 1;
        if (tile_ok) {
            uint64_t need = kLowMask;
            if (kind_has_target(gates[i].kind)) need |= uint64_t(1) << gates[i].target;
            uint64_t round_set = kind_has_target(gates[i].kind) ? (uint64_t(1) << gates[i].target) : 0;
            int rounds = 1;
            int diags = gates[i].kind == kKindDiagN;
            int pass_class = lean_first ? gate_class(gates[i], mats) : 2;
            while (j < count && j - i < kMaxPassGates) {
                const qs_gate& g = gates[j];
                if (g.kind == kKindDiagN && diags >= kMaxPassDiags) break;
                // passes of lean kinds stay on the lean kernels, passes of CNOTs
                // on k_perm (schedule_program's classes)
                if (lean_first && pass_class < 2 && gate_class(g, mats) != pass_class) break;
                diags += g.kind == kKindDiagN;
                uint64_t nn = need, rs = round_set;
                int nr = rounds;
                if (kind_has_target(g.kind)) {
                    uint64_t b = uint64_t(1) << g.target;
                    nn |= b;
                    if (!(rs & b)) {
                        if (__builtin_popcountll(rs) >= kRegLog2) {
                            rs = 0;
                            ++nr;
                        }
                        rs |= b;
                    }
                }
                if (__builtin_popcountll(nn) > kTileLog2 || nr > kMaxRounds) break;
                need = nn;
                round_set = rs;
                rounds = nr;
                ++j;
            }
        }
        out.push_back({i, j - i});
        i = j;
    }
    return out;
}

int validate_gate(const qs_state* st, const qs_gate& g, uint64_t mats_len, int num_edges) {
    const int n = st->n, m = st->m;
    uint64_t entry;
    if (g.kind == QS_KIND_1Q || g.kind == QS_KIND_CTRL) {
        if (g.target < 0 || g.target >= n)
            return fail(QS_ERR_VALUE, "qubit %d out of range for n=%d", g.target, n);
        if (g.target >= m)
            return fail(QS_ERR_LOCALITY,
                        "qubit %d is global for m=%d; route through the distribution module",
                        g.target, m);
        if (g.kind == QS_KIND_CTRL) {
            if (g.control == g.target) return fail(QS_ERR_VALUE, "control and target must differ");
            if (g.control < 0 || g.control >= n)
                return fail(QS_ERR_VALUE, "qubit %d out of range for n=%d", g.control, n);
            if (g.control >= m)
                return fail(QS_ERR_LOCALITY,
                            "both qubits must be local for the local controlled kernel");
        }
        entry = 8;
    } else if (g.kind == QS_KIND_CUTPHASE) {
        entry = 2 * uint64_t(num_edges + 1);
    } else {
        return fail(QS_ERR_VALUE, "unknown gate kind %d", g.kind);
    }
    uint64_t last = g.offset + uint64_t(st->num_states - 1) * g.stride + entry;
    if (last > mats_len)
        return fail(QS_ERR_VALUE, "gate table entry [%llu, %llu) beyond %llu doubles",
                    (unsigned long long)g.offset, (unsigned long long)last,
                    (unsigned long long)mats_len);
    return QS_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int qs_abi_version(void) { return QSB200_ABI_VERSION; }

const char* qs_last_error(void) { return g_last_error.c_str(); }

int qs_device_count(int32_t* out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *out = 0;
        return fail(QS_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    *out = n;
    return QS_OK;
}

uint64_t qs_host_sync_count(void) { return g_host_syncs.load(std::memory_order_relaxed); }

int qs_counters(const qs_state* st, uint64_t* messages, uint64_t* amplitudes) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    *messages = st->messages;
    *amplitudes = st->amplitudes;
    return QS_OK;
}

int qs_state_create(int32_t num_qubits, int32_t num_local_qubits, int32_t rank_index,
                    int32_t num_states, int32_t device, qs_state** out) {
    *out = nullptr;
    const int n = num_qubits, m = num_local_qubits;
    if (!(0 < m && m <= n))
        return fail(QS_ERR_VALUE, "need 0 < num_local_qubits <= num_qubits, got m=%d, n=%d", m, n);
    if (n > 62) return fail(QS_ERR_VALUE, "at most 62 qubits");
    if (!(0 <= rank_index && (uint64_t)rank_index < (uint64_t(1) << (n - m))))
        return fail(QS_ERR_VALUE, "rank_index %d out of range for %d rank bits", rank_index, n - m);
    if (num_states < 1) return fail(QS_ERR_VALUE, "need at least one state");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(QS_ERR_CUDA, "no CUDA device (%s); the B200 core has no CPU fallback",
                    cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(QS_ERR_VALUE, "device %d of %d", device, ndev);
    qs_state* st = new (std::nothrow) qs_state();
    if (!st) return fail(QS_ERR_NOMEM, "host allocation");
    st->n = n;
    st->m = m;
    st->rank = rank_index;
    st->num_states = num_states;
    st->device = device;
    st->amps_per_state = uint64_t(1) << m;
    int rc = QS_OK;
    do {
        if ((e = cudaSetDevice(device)) != cudaSuccess) break;
        if ((e = cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking)) != cudaSuccess) break;
        if ((e = cudaStreamCreateWithFlags(&st->comm_stream, cudaStreamNonBlocking)) != cudaSuccess)
            break;
        size_t bytes = sizeof(double2) * st->amps_per_state * size_t(num_states);
        if ((e = cudaMalloc(&st->psi, bytes)) != cudaSuccess) break;
        if ((e = cudaMalloc(&st->d_u, 8 * sizeof(double))) != cudaSuccess) break;
        for (auto& ev : st->ev)
            if ((e = cudaEventCreate(&ev)) != cudaSuccess) break;
        if (e != cudaSuccess) break;
        if ((e = cudaMemsetAsync(st->psi, 0, bytes, st->stream)) != cudaSuccess) break;
    } while (0);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // clear the (non-sticky) error before later launches
        rc = fail(e == cudaErrorMemoryAllocation ? QS_ERR_NOMEM : QS_ERR_CUDA,
                  "qs_state_create(n=%d, m=%d, states=%d): %s", n, m, num_states,
                  cudaGetErrorString(e));
        qs_state_destroy(st);
        return rc;
    }
    *out = st;
    return QS_OK;
}

int qs_state_destroy(qs_state* st) {
    if (!st) return QS_OK;
    cudaSetDevice(st->device);
    if (st->stream) host_sync_stream(st->stream);
    if (st->comm && g_nccl.loaded) g_nccl.CommDestroy(st->comm);
    for (auto& r : st->recs) cudaEventDestroy(r.start), cudaEventDestroy(r.stop);
    for (auto& ev : st->ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : st->sync_ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : st->nccl_ev)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : st->opened_ev) cudaEventDestroy(ev);
    cudaFree(st->psi);
    cudaFree(st->d_mats);
    cudaFree(st->d_pass);
    cudaFree(st->d_scratch);
    cudaFree(st->d_u);
    cudaFree(st->d_stage[0]);  // d_stage[1] points into the same allocation
    if (st->h_out) cudaFreeHost(st->h_out);
    if (st->stream) cudaStreamDestroy(st->stream);
    if (st->comm_stream) cudaStreamDestroy(st->comm_stream);
    delete st;
    return QS_OK;
}

int qs_state_info(const qs_state* st, int32_t* n, int32_t* m, int32_t* r, int32_t* ns,
                  uint64_t* aps) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    *n = st->n;
    *m = st->m;
    *r = st->rank;
    *ns = st->num_states;
    *aps = st->amps_per_state;
    return QS_OK;
}

int qs_state_device_ptr(const qs_state* st, void** out) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    *out = st->psi;
    return QS_OK;
}

int qs_synchronize(qs_state* st) {
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(host_sync_stream(st->stream));
    return QS_OK;
}

int qs_state_upload(qs_state* st, const double* host, uint64_t offset, uint64_t count) {
    if (int rc = ensure_device(st)) return rc;
    uint64_t total = st->amps_per_state * uint64_t(st->num_states);
    if (offset > total || count > total - offset)
        return fail(QS_ERR_VALUE, "upload range [%llu, +%llu) beyond %llu amplitudes",
                    (unsigned long long)offset, (unsigned long long)count,
                    (unsigned long long)total);
    if (count == 0) return QS_OK;
    CUDA_TRY(cudaMemcpyAsync(st->psi + offset, host, count * sizeof(double2),
                             cudaMemcpyHostToDevice, st->stream));
    CUDA_TRY(host_sync_stream(st->stream));
    return QS_OK;
}

int qs_state_download(qs_state* st, double* host, uint64_t offset, uint64_t count) {
    if (int rc = ensure_device(st)) return rc;
    uint64_t total = st->amps_per_state * uint64_t(st->num_states);
    if (offset > total || count > total - offset)
        return fail(QS_ERR_VALUE, "download range beyond the state");
    if (count == 0) return QS_OK;
    CUDA_TRY(cudaMemcpyAsync(host, st->psi + offset, count * sizeof(double2),
                             cudaMemcpyDeviceToHost, st->stream));
    CUDA_TRY(host_sync_stream(st->stream));
    return QS_OK;
}

// Full-duplex step boundary: read the whole slice into host_out while the
// next input streams in from host_in, chunk by chunk -- D2H of chunk i+1 runs
// on the comm stream while H2D of chunk i runs on the compute stream (PCIe is
// full duplex).  Chunk i is overwritten only after its own D2H completed.
int qs_state_exchange_host(qs_state* st, const double* host_in, double* host_out,
                           uint64_t chunk) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = ensure_device(st)) return rc;
    const uint64_t total = st->amps_per_state * uint64_t(st->num_states);
    if (chunk == 0) chunk = uint64_t(1) << 24;
    cudaEvent_t start, done;
    CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(start, st->stream));
    CUDA_TRY(cudaStreamWaitEvent(st->comm_stream, start, 0));
    std::vector<cudaEvent_t> evs;
    for (uint64_t off = 0; off < total; off += chunk) {
        const uint64_t len = std::min(chunk, total - off);
        CUDA_TRY(cudaMemcpyAsync(host_out + 2 * off, st->psi + off, len * sizeof(double2),
                                 cudaMemcpyDeviceToHost, st->comm_stream));
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(ev, st->comm_stream));
        evs.push_back(ev);
        CUDA_TRY(cudaStreamWaitEvent(st->stream, ev, 0));
        CUDA_TRY(cudaMemcpyAsync(st->psi + off, host_in + 2 * off, len * sizeof(double2),
                                 cudaMemcpyHostToDevice, st->stream));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(done, st->comm_stream));
    CUDA_TRY(cudaStreamWaitEvent(st->stream, done, 0));
    CUDA_TRY(host_sync_stream(st->stream));
    for (auto e : evs) cudaEventDestroy(e);
    cudaEventDestroy(start);
    cudaEventDestroy(done);
    return QS_OK;
}

int qs_init_zero(qs_state* st) {
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(cudaMemsetAsync(st->psi, 0,
                             sizeof(double2) * st->amps_per_state * size_t(st->num_states),
                             st->stream));
    return QS_OK;
}

int qs_init_basis(qs_state* st, uint64_t index) {
    if (int rc = ensure_device(st)) return rc;
    if (index >= (uint64_t(1) << st->n))
        return fail(QS_ERR_VALUE, "basis index %llu out of range for %d qubits",
                    (unsigned long long)index, st->n);
    if (int rc = qs_init_zero(st)) return rc;
    if ((index >> st->m) == uint64_t(st->rank)) {
        // stream-ordered, no host sync (a pool reset used to block ~2 ms here)
        launch_set_basis(st->psi, st->amps_per_state, uint64_t(st->num_states),
                         index & (st->amps_per_state - 1), st->stream);
        CUDA_TRY(cudaGetLastError());
    }
    return QS_OK;
}

int qs_init_constant(qs_state* st, double re, double im) {
    if (int rc = ensure_device(st)) return rc;
    launch_fill(st->psi, st->amps_per_state * uint64_t(st->num_states), make_double2(re, im),
                st->stream);
    CHECK_LAUNCH();
    return QS_OK;
}

int qs_init_gaussian(qs_state* st, uint64_t seed) {
    if (int rc = ensure_device(st)) return rc;
    launch_gaussian(st->psi, st->amps_per_state, st->num_states, uint64_t(st->rank) << st->m, seed,
                    st->stream);
    CHECK_LAUNCH();
    return QS_OK;
}

int qs_scale(qs_state* st, double factor) {
    if (int rc = ensure_device(st)) return rc;
    launch_scale(st->psi, st->amps_per_state * uint64_t(st->num_states), factor, st->stream);
    CHECK_LAUNCH();
    return QS_OK;
}

int qs_state_diff(qs_state* a, const qs_state* b, double* out) {
    if (!a || !b || !out) return fail(QS_ERR_VALUE, "null argument");
    if (a->device != b->device) return fail(QS_ERR_VALUE, "states on different devices");
    const uint64_t total = a->amps_per_state * uint64_t(a->num_states);
    if (total != b->amps_per_state * uint64_t(b->num_states))
        return fail(QS_ERR_VALUE, "states of different sizes");
    if (int rc = ensure_device(a)) return rc;
    if (int rc = grow(&a->d_scratch, &a->scratch_cap, 4)) return rc;
    // b's queued work first: a's stream waits for b's stream
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev, b->stream));
    CUDA_TRY(cudaStreamWaitEvent(a->stream, ev, 0));
    cudaEventDestroy(ev);
    launch_state_diff(a->psi, b->psi, total, a->d_scratch, a->stream);
    CHECK_LAUNCH();
    double h[4];
    CUDA_TRY(cudaMemcpyAsync(h, a->d_scratch, sizeof(h), cudaMemcpyDeviceToHost, a->stream));
    CUDA_TRY(host_sync_stream(a->stream));
    out[0] = h[0];
    out[1] = h[2];
    out[2] = h[3];
    out[3] = h[1];
    return QS_OK;
}

int qs_apply_diagonal(qs_state* st, const double* factors, uint64_t offset, uint64_t count) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = ensure_device(st)) return rc;
    const uint64_t total = st->amps_per_state * uint64_t(st->num_states);
    if (offset > total || count > total - offset)
        return fail(QS_ERR_VALUE, "diagonal range beyond the state");
    if (count == 0) return QS_OK;
    if (!factors) return fail(QS_ERR_VALUE, "factors is NULL");
    const uint64_t chunk = std::min<uint64_t>(count, uint64_t(1) << 22);
    if (int rc = grow(&st->d_scratch, &st->scratch_cap, size_t(2 * chunk))) return rc;
    for (uint64_t done = 0; done < count; done += chunk) {
        const uint64_t k = std::min(chunk, count - done);
        CUDA_TRY(cudaMemcpyAsync(st->d_scratch, factors + 2 * done, k * sizeof(double2),
                                 cudaMemcpyHostToDevice, st->stream));
        launch_mul_factors(st->psi + offset + done, reinterpret_cast<const double2*>(st->d_scratch),
                           k, st->stream);
        CHECK_LAUNCH();
    }
    // the host buffer may be released when we return
    CUDA_TRY(host_sync_stream(st->stream));
    return QS_OK;
}

namespace {
// const_in: every amplitude of the state is (re, im) before the program (the
// first pass generates it or a fill precedes it); nullptr: the state as it is.
int apply_program_impl(qs_state* st, const qs_gate* gates, int32_t count, const double* mats,
                       uint64_t mats_len, const int32_t* edges, int32_t num_edges, int32_t fuse,
                       const double* const_in) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (count < 0) return fail(QS_ERR_VALUE, "negative gate count");
    if (count == 0) {
        st->last_passes = 0;
        if (const_in) return qs_init_constant(st, const_in[0], const_in[1]);
        return QS_OK;
    }
    if (int rc = ensure_device(st)) return rc;
    CutTerms ct;
    bool has_phase = false;
    for (int i = 0; i < count; ++i) has_phase |= gates[i].kind == QS_KIND_CUTPHASE;
    if (has_phase) {
        if (int rc = build_cut_terms(edges, num_edges, st->n, &ct)) return rc;
    } else {
        memset(&ct, 0, sizeof(ct));
        num_edges = 0;
    }
    for (int i = 0; i < count; ++i)
        if (int rc = validate_gate(st, gates[i], mats_len, num_edges)) return rc;
    static thread_local FactoredProgram fp;
    static thread_local std::vector<double> all;
    // QSB_DEBUG_TIME: host time of each phase on stderr
    static const bool dbg_time = getenv("QSB_DEBUG_TIME") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t_start = now(), t_factor = t_start, t_upload = t_start, t_fp = t_start;
    bool lean_first = false;
    if (fuse == QS_FUSE_FACTORED && st->m >= kTileLog2) {
        // rewrite, then plan the rewritten program; its parameters and diagonal
        // tables follow the caller's table in one upload.  Programs where fewer
        // than half of the gates factor (noise trajectories) run exact: the
        // rewrite does not pay there.
        uint64_t support = 0;
        for (int e = 0; e < 2 * num_edges; ++e) support |= uint64_t(1) << edges[e];
        // large states: an extra pass costs less than moving a lean pass to k_tile
        // (QSB_LEAN_FIRST_M moves the threshold; read per call so tests can set it)
        const char* lf = getenv("QSB_LEAN_FIRST_M");
        lean_first = st->m >= (lf ? atoi(lf) : 24);
        factor_program(gates, count, mats, mats_len, st->m, st->num_states, num_edges, support, &fp,
                       lean_first);
        t_fp = now();
        // CNOTs count as factored: their passes run as permutations (k_perm), so a
        // program of CNOTs between two exchanges does not fall back to k_tile
        int cnots = 0;
        if (st->num_states == 1 && st->m > 13)
            for (int i = 0; i < count; ++i) cnots += gate_is_cnot(gates[i], mats);
        if (2 * (fp.factored + cnots) >= count) {
            all.assign(mats, mats + mats_len);
            all.insert(all.end(), fp.extra.begin(), fp.extra.end());
            static const bool reorder = getenv("QSB_NO_REORDER") == nullptr;
            if (reorder)
                schedule_program(fp.gates, st->m, support, all.data(), st->num_states, lean_first);
            g_zero_off = fp.zero_off;
            g_factored = true;
            gates = fp.gates.data();
            count = int(fp.gates.size());
            mats = all.data();
            mats_len = all.size();
        } else {
            lean_first = false;  // the program runs exact: the plain planner
        }
    }
    struct FactoredScope {  // cleared on every exit
        ~FactoredScope() { g_factored = false; }
    } factored_scope;
    t_factor = now();
    if (int rc = grow(&st->d_mats, &st->mats_cap, mats_len ? mats_len : 1)) return rc;
    if (mats_len)
        CUDA_TRY(cudaMemcpyAsync(st->d_mats, mats, mats_len * sizeof(double),
                                 cudaMemcpyHostToDevice, st->stream));
    t_upload = now();
    std::vector<PassPlan> plan = plan_passes(gates, count, st->m, fuse != 0, lean_first, mats);
    int passes = 0;
    if (const_in)
        g_const_in = {true, make_double2(const_in[0], const_in[1]),
                      st->amps_per_state * uint64_t(st->num_states)};
    for (size_t pi = 0; pi < plan.size(); ++pi) {
        const PassPlan& pp = plan[pi];
        // the internal kinds of a factored program only exist as tile-pass gates
        const bool single = pp.count == 1 && gates[pp.first].kind <= QS_KIND_CUTPHASE;
        // a CNOT pass right behind a lean pass: offered to the lean launcher,
        // which folds it into its copy-out when the tile holds every target
        g_absorb.count = 0;
        g_absorb.done = false;
        if (g_factored && !single && pi + 1 < plan.size() && st->num_states == 1 &&
            gate_class(gates[pp.first], mats) == 0) {
            const PassPlan& nx = plan[pi + 1];
            bool all_cnot = nx.count <= kMaxPassGates;
            for (int i = 0; i < nx.count && all_cnot; ++i)
                all_cnot = gate_is_cnot(gates[nx.first + i], mats);
            for (int i = 0; i < pp.count && all_cnot; ++i)
                all_cnot = kind_is_lean(gates[pp.first + i].kind);
            if (all_cnot) {
                g_absorb.count = nx.count;
                for (int i = 0; i < nx.count; ++i) {
                    g_absorb.controls[i] = gates[nx.first + i].control;
                    g_absorb.targets[i] = gates[nx.first + i].target;
                }
            }
        }
        if (single && g_const_in.on) {  // the streaming kernels read their input from HBM
            launch_fill(st->psi, g_const_in.total, g_const_in.v, st->stream);
            g_const_in.on = false;
        }
        int rc = single ? launch_single(st, gates[pp.first], ct, mats)
                        : launch_tile(st, gates, pp.first, pp.count, ct, mats);
        if (rc) {
            g_const_in.on = false;
            g_absorb.count = 0;
            return rc;
        }
        ++passes;
        if (g_absorb.done) ++pi;  // the CNOT pass ran inside this one
        g_absorb.count = 0;
        g_absorb.done = false;
    }
    st->last_passes = passes;
    if (dbg_time) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t_end = now();
        fprintf(stderr, "qs_apply_program: %d gates, %d passes, %.1f KB tables: factor %.3f ms, "
                "schedule %.3f ms, upload %.3f ms, plan+launch %.3f ms\n", count, passes,
                mats_len * 8.0 / 1024, ms(t_start, t_fp), ms(t_fp, t_factor), ms(t_factor, t_upload),
                ms(t_upload, t_end));
    }
    // no host sync: pageable H2D copies are staged before cudaMemcpyAsync returns,
    // so the caller may reuse `mats`, and the device tables are stream-ordered.
    return QS_OK;
}
}  // namespace

int qs_apply_program(qs_state* st, const qs_gate* gates, int32_t count, const double* mats,
                     uint64_t mats_len, const int32_t* edges, int32_t num_edges, int32_t fuse) {
    return apply_program_impl(st, gates, count, mats, mats_len, edges, num_edges, fuse, nullptr);
}

int qs_apply_program_on_constant(qs_state* st, double re, double im, const qs_gate* gates,
                                 int32_t count, const double* mats, uint64_t mats_len,
                                 const int32_t* edges, int32_t num_edges, int32_t fuse) {
    const double c[2] = {re, im};
    return apply_program_impl(st, gates, count, mats, mats_len, edges, num_edges, fuse, c);
}

// Planning only (no device needed): writes the first gate index of every
// pass into starts[] (up to cap) and the pass count into *npasses.
int qs_plan_program(int32_t num_local_qubits, const qs_gate* gates, int32_t count, int32_t fuse,
                    int32_t* starts, int32_t cap, int32_t* npasses) {
    if (count < 0 || num_local_qubits < 1) return fail(QS_ERR_VALUE, "bad plan arguments");
    for (int i = 0; i < count; ++i)
        if (gates[i].kind != QS_KIND_CUTPHASE &&
            (gates[i].target < 0 || gates[i].target >= num_local_qubits))
            return fail(QS_ERR_VALUE, "target %d outside the local qubits", gates[i].target);
    std::vector<PassPlan> plan = plan_passes(gates, count, num_local_qubits, fuse != 0);
    for (size_t k = 0; k < plan.size() && (int)k < cap; ++k) starts[k] = plan[k].first;
    *npasses = (int32_t)plan.size();
    return QS_OK;
}

int qs_decompose_2x2(const double* u, double* out) {
    if (!u || !out) return fail(QS_ERR_VALUE, "null argument");
    if (!decompose_2x2(u, out)) return fail(QS_ERR_VALUE, "not a non-diagonal unitary");
    return QS_OK;
}

int qs_last_program_passes(const qs_state* st, int32_t* passes) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    *passes = st->last_passes;
    return QS_OK;
}

int qs_apply_1q(qs_state* st, int32_t q, const double* u, uint64_t u_stride) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (q < 0) return fail(QS_ERR_VALUE, "negative qubit index");
    qs_gate g{QS_KIND_1Q, q, -1, 0, 0, u_stride};
    uint64_t len = u_stride ? u_stride * uint64_t(st->num_states - 1) + 8 : 8;
    return qs_apply_program(st, &g, 1, u, len, nullptr, 0, 0);
}

int qs_apply_controlled(qs_state* st, int32_t control, int32_t target, const double* u,
                        uint64_t u_stride) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    qs_gate g{QS_KIND_CTRL, target, control, 0, 0, u_stride};
    uint64_t len = u_stride ? u_stride * uint64_t(st->num_states - 1) + 8 : 8;
    return qs_apply_program(st, &g, 1, u, len, nullptr, 0, 0);
}

int qs_apply_cut_phase(qs_state* st, const int32_t* edges, int32_t num_edges, const double* lut,
                       uint64_t lut_stride) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    qs_gate g{QS_KIND_CUTPHASE, 0, -1, 0, 0, lut_stride};
    uint64_t entry = 2 * uint64_t(num_edges + 1);
    uint64_t len = lut_stride ? lut_stride * uint64_t(st->num_states - 1) + entry : entry;
    return qs_apply_program(st, &g, 1, lut, len, edges, num_edges, 0);
}

int qs_observable(qs_state* st, int32_t kind, int32_t q, const int32_t* edges, int32_t num_edges,
                  double* out) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = ensure_device(st)) return rc;
    CutTerms ct;
    memset(&ct, 0, sizeof(ct));
    if (kind == QS_OBS_PROB || kind == QS_OBS_Z) {
        if (q < 0 || q >= st->n) return fail(QS_ERR_VALUE, "qubit %d out of range", q);
    } else if (kind == QS_OBS_MAXCUT) {
        if (int rc = build_cut_terms(edges, num_edges, st->n, &ct)) return rc;
    } else if (kind != QS_OBS_NORM) {
        return fail(QS_ERR_VALUE, "unknown observable %d", kind);
    }
    int eff_kind = kind;
    bool zero = false;
    if (kind == QS_OBS_PROB && q >= st->m) {
        // statevector.py:225-228: a global qubit selects the whole slice or nothing
        if ((st->rank >> (q - st->m)) & 1)
            eff_kind = QS_OBS_NORM;
        else
            zero = true;
    }
    if (zero) {
        for (int s = 0; s < st->num_states; ++s) out[s] = 0.0;
        return QS_OK;
    }
    size_t need = reduce_scratch_doubles(st->m, st->num_states) + st->num_states;
    if (int rc = grow(&st->d_scratch, &st->scratch_cap, need)) return rc;
    if (st->h_out_cap < size_t(st->num_states)) {
        if (st->h_out) cudaFreeHost(st->h_out);
        st->h_out = nullptr;
        CUDA_TRY(cudaMallocHost(&st->h_out, sizeof(double) * st->num_states));
        st->h_out_cap = st->num_states;
    }
    double* out_dev = st->d_scratch + reduce_scratch_doubles(st->m, st->num_states);
    {
        LaunchScope ls(st, kLaunchReduce);
        launch_observable(st->psi, st->m, st->num_states, eff_kind, q, uint64_t(st->rank) << st->m,
                          ct, st->d_scratch, out_dev, st->stream);
    }
    CHECK_LAUNCH();
    CUDA_TRY(cudaMemcpyAsync(st->h_out, out_dev, sizeof(double) * st->num_states,
                             cudaMemcpyDeviceToHost, st->stream));
    CUDA_TRY(host_sync_stream(st->stream));
    memcpy(out, st->h_out, sizeof(double) * st->num_states);
    return QS_OK;
}

// Host-side 2x2 products for noise matrices (qsb200.h; noise.py:70-80).
static inline __attribute__((always_inline)) void compose_one(const double* x, const double* y,
                                                              double* out) {
    double z[8];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double ar0 = x[4 * i + 0], ai0 = x[4 * i + 1];
            const double ar1 = x[4 * i + 2], ai1 = x[4 * i + 3];
            const double br0 = y[2 * j + 0], bi0 = y[2 * j + 1];
            const double br1 = y[4 + 2 * j], bi1 = y[4 + 2 * j + 1];
            double re = __builtin_fma(ar0, br0, 0.0);
            re = __builtin_fma(-ai0, bi0, re);
            re = __builtin_fma(ar1, br1, re);
            re = __builtin_fma(-ai1, bi1, re);
            double im = __builtin_fma(ar0, bi0, 0.0);
            im = __builtin_fma(ai0, br0, im);
            im = __builtin_fma(ar1, bi1, im);
            im = __builtin_fma(ai1, br1, im);
            z[4 * i + 2 * j] = re;
            z[4 * i + 2 * j + 1] = im;
        }
    memcpy(out, z, sizeof z);
}

// same loop with hardware FMA instructions inlined (fma is exact either way)
__attribute__((target("fma"))) static void compose_hw(const double* a, const double* b,
                                                      int64_t count, double* out) {
    for (int64_t s = 0; s < count; ++s) compose_one(a + 8 * s, b + 8 * s, out + 8 * s);
}

static void compose_sw(const double* a, const double* b, int64_t count, double* out) {
    for (int64_t s = 0; s < count; ++s) compose_one(a + 8 * s, b + 8 * s, out + 8 * s);
}

int qs_compose_2x2(const double* a, const double* b, int64_t count, double* out) {
    if (count < 0 || (count && (!a || !b || !out))) return fail(QS_ERR_VALUE, "bad compose args");
    if (__builtin_cpu_supports("fma")) compose_hw(a, b, count, out);
    else compose_sw(a, b, count, out);
    return QS_OK;
}

// Philox4x64-10 blocks for the noise streams (qsb200.h).
int qs_philox4x64(const uint64_t* keys, const uint64_t* ctr, int64_t count, uint64_t* out) {
    if (count < 0 || (count && (!keys || !ctr || !out))) return fail(QS_ERR_VALUE, "bad philox args");
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    for (int64_t i = 0; i < count; ++i) {
        uint64_t k0 = keys[2 * i], k1 = keys[2 * i + 1];
        uint64_t v0 = ctr[2 * i], v1 = ctr[2 * i + 1], v2 = 0, v3 = 0;
        for (int r = 0; r < 10; ++r) {
            if (r) { k0 += W0; k1 += W1; }
            const unsigned __int128 p0 = (unsigned __int128)M0 * v0;
            const unsigned __int128 p1 = (unsigned __int128)M1 * v2;
            const uint64_t hi0 = uint64_t(p0 >> 64), lo0 = uint64_t(p0);
            const uint64_t hi1 = uint64_t(p1 >> 64), lo1 = uint64_t(p1);
            v0 = hi1 ^ v1 ^ k0;
            v1 = lo1;
            v2 = hi0 ^ v3 ^ k1;
            v3 = lo0;
        }
        out[4 * i] = v0; out[4 * i + 1] = v1; out[4 * i + 2] = v2; out[4 * i + 3] = v3;
    }
    return QS_OK;
}

// All per-qubit probabilities P(q=1) of every state in one pass over the slice
// (cmd_run's "prob q" report, cli.py:161-172): out[num_states * n], each value
// identical to qs_observable(QS_OBS_PROB, q).
int qs_marginals(qs_state* st, double* out) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = ensure_device(st)) return rc;
    const int n = st->n, m = st->m, S = st->num_states;
    if (m < 12) {  // small slices: one reduction per qubit
        std::vector<double> tmp(S);
        for (int q = 0; q < n; ++q) {
            if (int rc = qs_observable(st, QS_OBS_PROB, q, nullptr, 0, tmp.data())) return rc;
            for (int s = 0; s < S; ++s) out[size_t(s) * n + q] = tmp[s];
        }
        return QS_OK;
    }
    size_t need = marginal_scratch_doubles(m, S) + size_t(S) * m + size_t(S);
    if (int rc = grow(&st->d_scratch, &st->scratch_cap, need)) return rc;
    double* dev_out = st->d_scratch + marginal_scratch_doubles(m, S);
    {
        LaunchScope ls(st, kLaunchReduce);
        launch_marginals(st->psi, m, S, st->d_scratch, dev_out, st->stream);
    }
    CHECK_LAUNCH();
    std::vector<double> local(size_t(S) * m);
    CUDA_TRY(cudaMemcpyAsync(local.data(), dev_out, sizeof(double) * local.size(),
                             cudaMemcpyDeviceToHost, st->stream));
    CUDA_TRY(host_sync_stream(st->stream));
    std::vector<double> norms;
    if (n > m) {  // global qubits: the whole slice or nothing (statevector.py:225-228)
        norms.resize(S);
        if (int rc = qs_observable(st, QS_OBS_NORM, 0, nullptr, 0, norms.data())) return rc;
    }
    for (int s = 0; s < S; ++s)
        for (int q = 0; q < n; ++q) {
            double v;
            if (q < m) {
                // device layout: [S][11] for q < 11, then [S][m-11] for q >= 11
                v = q < 11 ? local[size_t(s) * 11 + q]
                           : local[size_t(S) * 11 + size_t(s) * (m - 11) + (q - 11)];
            } else {
                v = ((st->rank >> (q - m)) & 1) ? norms[s] : 0.0;
            }
            out[size_t(s) * n + q] = v;
        }
    return QS_OK;
}

// ---- global-qubit path --------------------------------------------------------
// A partner slice on another device of this process (thread-per-rank over
// several GPUs) needs peer access from ours; IPC-mapped slices of other
// processes already have it (cudaIpcMemLazyEnablePeerAccess).
static int ensure_peer_access(qs_state* st, const void* peer) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, peer) != cudaSuccess) {
        (void)cudaGetLastError();
        return QS_OK;  // not a pointer the runtime knows: let the kernel report it
    }
    if (attr.type != cudaMemoryTypeDevice || attr.device == st->device) return QS_OK;
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, st->device, attr.device));
    if (!can)
        return fail(QS_ERR_COMM, "device %d cannot access device %d's memory (no P2P)",
                    st->device, attr.device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(attr.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(QS_ERR_COMM, "cudaDeviceEnablePeerAccess(%d): %s", attr.device,
                    cudaGetErrorString(e));
    (void)cudaGetLastError();
    return QS_OK;
}

int qs_exchange_gate_peer(qs_state* st, void* peer_amps, int32_t is_lower, const double* u,
                          int32_t control_local) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (!peer_amps) return fail(QS_ERR_VALUE, "null peer pointer");
    if (st->num_states != 1) return fail(QS_ERR_VALUE, "exchange needs a single-state handle");
    if (control_local >= st->m) return fail(QS_ERR_LOCALITY, "control %d is not local", control_local);
    if (int rc = ensure_device(st)) return rc;
    if (int rc = ensure_peer_access(st, peer_amps)) return rc;
    CUDA_TRY(cudaMemcpyAsync(st->d_u, u, 8 * sizeof(double), cudaMemcpyHostToDevice, st->stream));
    {
        LaunchScope ls(st, kLaunchExchange);
        launch_exchange_peer(st->psi, reinterpret_cast<double2*>(peer_amps), st->m, is_lower != 0,
                             st->d_u, control_local, st->stream);
    }
    CHECK_LAUNCH();
    // accounting in TransportCounters terms: one transfer out and one back,
    // 2 * 2^(m-1) amplitudes leave this rank (reads by the partner + writes to it)
    uint64_t moved = st->amps_per_state >> (control_local >= 0 ? 1 : 0);
    st->messages += 2;
    st->amplitudes += moved;
    // no host sync: the caller orders the partner's work with qs_sync_event*
    return QS_OK;
}

int qs_swap_qubits_peer(qs_state* st, void* peer_amps, int32_t local_qubit, int32_t rank_bit) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (!peer_amps) return fail(QS_ERR_VALUE, "null peer pointer");
    if (st->num_states != 1) return fail(QS_ERR_VALUE, "swap needs a single-state handle");
    if (local_qubit < 0 || local_qubit >= st->m)
        return fail(QS_ERR_LOCALITY, "qubit %d is not local", local_qubit);
    if (int rc = ensure_device(st)) return rc;
    if (int rc = ensure_peer_access(st, peer_amps)) return rc;
    {
        LaunchScope ls(st, kLaunchExchange);
        launch_swap_peer(st->psi, reinterpret_cast<double2*>(peer_amps), st->m, local_qubit,
                         rank_bit ? 1 : 0, st->stream);
    }
    CHECK_LAUNCH();
    st->messages += 2;
    st->amplitudes += st->amps_per_state >> 1;
    return QS_OK;
}

int qs_swap_qubits_local(qs_state* st, int32_t a, int32_t c) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (a == c) return fail(QS_ERR_VALUE, "swap needs two different qubits");
    if (a < 0 || c < 0 || a >= st->m || c >= st->m)
        return fail(QS_ERR_LOCALITY, "both qubits must be local");
    if (int rc = ensure_device(st)) return rc;
    {
        LaunchScope ls(st, kLaunchExchange);
        launch_swap_local(st->psi, st->m, st->num_states, a, c, st->stream);
    }
    CHECK_LAUNCH();
    return QS_OK;
}

int qs_state_ipc_handle(const qs_state* st, unsigned char* handle64) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    CUDA_TRY(cudaSetDevice(st->device));
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, st->psi));
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle64, &h, 64);
    return QS_OK;
}

int qs_peer_open(qs_state* st, const unsigned char* handle64, void** peer_amps) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    CUDA_TRY(cudaSetDevice(st->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(peer_amps, h, cudaIpcMemLazyEnablePeerAccess));
    return QS_OK;
}

int qs_peer_close(qs_state* st, void* peer_amps) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    CUDA_TRY(cudaSetDevice(st->device));
    CUDA_TRY(cudaIpcCloseMemHandle(peer_amps));
    return QS_OK;
}

int qs_nccl_unique_id(unsigned char* id128) {
    if (int rc = nccl_load()) return rc;
    NcclId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    memcpy(id128, id.internal, 128);
    return QS_OK;
}

int qs_comm_init(qs_state* st, const unsigned char* id128, int32_t nranks, int32_t rank) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = nccl_load()) return rc;
    if (int rc = ensure_device(st)) return rc;
    NcclId id;
    memcpy(id.internal, id128, 128);
    NCCL_TRY(g_nccl.CommInitRank(&st->comm, nranks, id, rank));
    return QS_OK;
}

int qs_comm_destroy(qs_state* st) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (st->comm && g_nccl.loaded) {
        ensure_device(st);
        NCCL_TRY(g_nccl.CommDestroy(st->comm));
    }
    st->comm = nullptr;
    return QS_OK;
}

// The reference's three-step scheme (distribution.py:121-178) as a pipelined
// NCCL exchange: chunk k goes out and comes back on the comm stream while the
// compute stream updates chunk k-1; updated halves land in place in the
// outbound half, which is what lets the pipeline run without a half-state
// receive buffer.
int qs_exchange_gate_nccl(qs_state* st, int32_t peer, int32_t is_lower, const double* u,
                          int32_t control_local, uint64_t chunk) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (!st->comm) return fail(QS_ERR_COMM, "qs_comm_init was not called");
    if (st->num_states != 1) return fail(QS_ERR_VALUE, "exchange needs a single-state handle");
    if (chunk == 0) return fail(QS_ERR_VALUE, "chunk must be positive");
    if (control_local >= st->m) return fail(QS_ERR_LOCALITY, "control %d is not local", control_local);
    if (int rc = ensure_device(st)) return rc;
    const uint64_t half = st->amps_per_state / 2;
    const uint64_t c = std::min<uint64_t>(chunk, half);
    // one allocation holds both staging chunks, so they always grow together
    if (int rc = grow(&st->d_stage[0], &st->stage_cap, 2 * c)) return rc;
    st->d_stage[1] = st->d_stage[0] + st->stage_cap / 2;
    CUDA_TRY(cudaMemcpyAsync(st->d_u, u, 8 * sizeof(double), cudaMemcpyHostToDevice, st->stream));
    double2* mine = is_lower ? st->psi : st->psi + half;
    double2* outbound = is_lower ? st->psi + half : st->psi;
    const uint64_t mine_first = is_lower ? 0 : half;
    const uint64_t nchunks = (half + c - 1) / c;
    // the pipeline's events live with the handle (created on first use)
    for (auto& ev : st->nccl_ev)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaEvent_t* ev_in = st->nccl_ev;
    cudaEvent_t* ev_done = st->nccl_ev + 2;
    cudaEvent_t ev_start = st->nccl_ev[4], ev_end = st->nccl_ev[5];
    CUDA_TRY(cudaEventRecord(ev_start, st->stream));
    CUDA_TRY(cudaStreamWaitEvent(st->comm_stream, ev_start, 0));
    const size_t dbl = 2;  // doubles per amplitude
    for (uint64_t k = 0; k <= nchunks; ++k) {
        // comm: send chunk k out / receive partner's chunk k; return chunk k-1
        if (k > 0) CUDA_TRY(cudaStreamWaitEvent(st->comm_stream, ev_done[(k - 1) & 1], 0));
        NCCL_TRY(g_nccl.GroupStart());
        if (k < nchunks) {
            uint64_t len = std::min(c, half - k * c);
            NCCL_TRY(g_nccl.Send(outbound + k * c, len * dbl, kNcclFloat64, peer, st->comm,
                                 st->comm_stream));
            NCCL_TRY(g_nccl.Recv(st->d_stage[k & 1], len * dbl, kNcclFloat64, peer, st->comm,
                                 st->comm_stream));
            st->messages += 1;
            st->amplitudes += len;
        }
        if (k > 0) {
            uint64_t len = std::min(c, half - (k - 1) * c);
            NCCL_TRY(g_nccl.Send(st->d_stage[(k - 1) & 1], len * dbl, kNcclFloat64, peer, st->comm,
                                 st->comm_stream));
            NCCL_TRY(g_nccl.Recv(outbound + (k - 1) * c, len * dbl, kNcclFloat64, peer, st->comm,
                                 st->comm_stream));
            st->messages += 1;
            st->amplitudes += len;
        }
        NCCL_TRY(g_nccl.GroupEnd());
        if (k < nchunks) {
            CUDA_TRY(cudaEventRecord(ev_in[k & 1], st->comm_stream));
            // compute: pair update of chunk k (mine[k], partner's chunk in stage)
            CUDA_TRY(cudaStreamWaitEvent(st->stream, ev_in[k & 1], 0));
            uint64_t len = std::min(c, half - k * c);
            double2* a = is_lower ? mine + k * c : st->d_stage[k & 1];
            double2* b = is_lower ? st->d_stage[k & 1] : mine + k * c;
            {
                LaunchScope ls(st, kLaunchExchange);
                launch_pair_update_halves(a, b, len, mine_first + k * c, st->d_u, control_local,
                                          st->stream);
            }
            CHECK_LAUNCH();
            CUDA_TRY(cudaEventRecord(ev_done[k & 1], st->stream));
        }
    }
    CUDA_TRY(cudaEventRecord(ev_end, st->comm_stream));
    CUDA_TRY(cudaStreamWaitEvent(st->stream, ev_end, 0));
    // stream-ordered: the next kernels on st->stream follow the exchange
    return QS_OK;
}

// ---- cross-rank ordering without host syncs ---------------------------------
namespace {
int make_sync_events(qs_state* st) {
    // the partner's thread may ask for them while this rank records one
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& ev : st->sync_ev)
        if (!ev)
            CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
    return QS_OK;
}
}  // namespace

int qs_sync_event(qs_state* st, int32_t which, void** ev) {
    if (!st || !ev) return fail(QS_ERR_VALUE, "null argument");
    if (which < 0 || which > 1) return fail(QS_ERR_VALUE, "sync event %d out of range", which);
    if (int rc = ensure_device(st)) return rc;
    if (int rc = make_sync_events(st)) return rc;
    *ev = reinterpret_cast<void*>(st->sync_ev[which]);
    return QS_OK;
}

int qs_sync_event_ipc(qs_state* st, int32_t which, unsigned char* handle64) {
    if (!st || !handle64) return fail(QS_ERR_VALUE, "null argument");
    if (which < 0 || which > 1) return fail(QS_ERR_VALUE, "sync event %d out of range", which);
    if (int rc = ensure_device(st)) return rc;
    if (int rc = make_sync_events(st)) return rc;
    cudaIpcEventHandle_t h;
    CUDA_TRY(cudaIpcGetEventHandle(&h, st->sync_ev[which]));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, 64);
    return QS_OK;
}

int qs_sync_event_open(qs_state* st, const unsigned char* handle64, void** ev) {
    if (!st || !handle64 || !ev) return fail(QS_ERR_VALUE, "null argument");
    if (int rc = ensure_device(st)) return rc;
    cudaIpcEventHandle_t h;
    memcpy(&h, handle64, 64);
    cudaEvent_t e;
    CUDA_TRY(cudaIpcOpenEventHandle(&e, h));
    st->opened_ev.push_back(e);
    *ev = reinterpret_cast<void*>(e);
    return QS_OK;
}

int qs_sync_event_record(qs_state* st, int32_t which) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (which < 0 || which > 1) return fail(QS_ERR_VALUE, "sync event %d out of range", which);
    if (int rc = ensure_device(st)) return rc;
    if (int rc = make_sync_events(st)) return rc;
    CUDA_TRY(cudaEventRecord(st->sync_ev[which], st->stream));
    return QS_OK;
}

int qs_stream_wait_event(qs_state* st, void* ev) {
    if (!st || !ev) return fail(QS_ERR_VALUE, "null argument");
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(cudaStreamWaitEvent(st->stream, reinterpret_cast<cudaEvent_t>(ev), 0));
    return QS_OK;
}

int qs_stream_busy(qs_state* st, int32_t* busy) {
    if (!st || !busy) return fail(QS_ERR_VALUE, "null argument");
    if (int rc = ensure_device(st)) return rc;
    cudaError_t e = cudaStreamQuery(st->stream);
    if (e == cudaErrorNotReady) {
        *busy = 1;
        return QS_OK;
    }
    CUDA_TRY(e);
    *busy = 0;
    return QS_OK;
}

// Debug builds (-DQSB_PROF): cycle counters of the tile kernel's phases.
int qs_debug_prof(unsigned long long* out8) { return prof_read(out8) ? QS_OK : QS_ERR_VALUE; }

// ---- timing ------------------------------------------------------------------
int qs_event_record(qs_state* st, int32_t slot) {
    if (!st || slot < 0 || slot >= 8) return fail(QS_ERR_VALUE, "bad event slot");
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(cudaEventRecord(st->ev[slot], st->stream));
    return QS_OK;
}

int qs_event_elapsed_ms(qs_state* st, int32_t a, int32_t b, float* ms) {
    if (!st || a < 0 || a >= 8 || b < 0 || b >= 8) return fail(QS_ERR_VALUE, "bad event slot");
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(host_sync_event(st->ev[b]));
    CUDA_TRY(cudaEventElapsedTime(ms, st->ev[a], st->ev[b]));
    return QS_OK;
}

int qs_launch_log(qs_state* st, int32_t enable) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    st->launch_log = enable != 0;
    return QS_OK;
}

// Read (and clear) the per-launch log: kind codes 1 gate1q, 2 controlled,
// 3 cut-phase, 4 tile pass, 5 exchange, 6 reduction.
int qs_launch_log_read(qs_state* st, float* ms, int32_t* kinds, int32_t cap, int32_t* count) {
    if (!st) return fail(QS_ERR_VALUE, "null state");
    if (int rc = ensure_device(st)) return rc;
    CUDA_TRY(host_sync_stream(st->stream));
    int k = 0;
    for (auto& r : st->recs) {
        if (k < cap) {
            float t = 0;
            cudaEventElapsedTime(&t, r.start, r.stop);
            ms[k] = t;
            kinds[k] = r.kind;
        }
        ++k;
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    st->recs.clear();
    *count = k;
    return QS_OK;
}

}  // extern "C"
