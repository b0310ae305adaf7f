// Global-qubit gate kernels (reference: distribution._exchange_pairs,
// distribution.py:121-178, Fig. 3 of the paper).
//
// For a gate on global qubit q the pairs are (lower rank, offset o) and
// (upper rank, offset o) for every local offset o.  k_exchange_peer is the
// fused compute+transfer kernel: each of the two partner ranks takes half of
// the pairs (split on a local bit that is not the control), loads its own
// member from local HBM and the partner's over NVLink (peer pointer), applies
// the 2x2, and stores both members back -- one of them into the partner's
// memory.  The transfer therefore overlaps the arithmetic load by load, with
// no staging buffer and no second phase.
//
// k_pair_halves is the step-2 compute of the reference's three-step scheme on
// a received chunk (used by the NCCL send/recv path in capi.cu).
#include "common.cuh"

namespace qsb {
namespace {

constexpr int kThreads = 256;
constexpr int kIlp = 4;

__global__ void __launch_bounds__(kThreads)
    k_exchange_peer(double2* __restrict__ mine, double2* __restrict__ peer, int m, int split_bit,
                    int is_lower, int control, uint64_t total, const double* __restrict__ u_dev) {
    double2 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = reinterpret_cast<const double2*>(u_dev)[k];
    double2* lower = is_lower ? mine : peer;
    double2* upper = is_lower ? peer : mine;
    const uint64_t side = uint64_t(is_lower ? 0 : 1) << split_bit;
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    uint64_t off[kIlp];
    double2 a[kIlp], b[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t j = first + uint64_t(i) * kThreads;
        if (j < total) {
            uint64_t o;
            if (split_bit < 0) {  // m == 1 with a local control: the lower rank owns the pair
                o = (control < 0) ? j : (insert0(j, control) | (uint64_t(1) << control));
            } else if (control < 0) {
                o = insert0(j, split_bit) | side;
            } else {
                int lb = control < split_bit ? control : split_bit;
                int hb = control < split_bit ? split_bit : control;
                o = insert0(insert0(j, lb), hb) | side | (uint64_t(1) << control);
            }
            off[i] = o;
            a[i] = lower[o];
            b[i] = upper[o];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t j = first + uint64_t(i) * kThreads;
        if (j < total) {
            pair_update(a[i], b[i], u);
            lower[off[i]] = a[i];
            upper[off[i]] = b[i];
        }
    }
}

// a[k], b[k] are the two members of pair k of a chunk; `first_offset` is the
// local offset of element 0 of the chunk on the lower rank (control test).
__global__ void __launch_bounds__(kThreads)
    k_pair_halves(double2* __restrict__ a, double2* __restrict__ b, uint64_t count,
                  uint64_t first_offset, int control, const double* __restrict__ u_dev) {
    double2 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = reinterpret_cast<const double2*>(u_dev)[k];
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += uint64_t(gridDim.x) * blockDim.x) {
        if (control >= 0 && !(((first_offset + k) >> control) & 1)) continue;
        double2 x = a[k], y = b[k];
        pair_update(x, y, u);
        a[k] = x;
        b[k] = y;
    }
}

// SWAP of physical qubits p (global: this rank's bit value b) and l (local)
// between partner ranks: the amplitude at local offset o with bit l = 1-b
// trades places with the partner's amplitude at o ^ 2^l.  Pure data movement;
// the two ranks split the pairs on local bit s (!= l).
__global__ void __launch_bounds__(kThreads)
    k_swap_peer(double2* __restrict__ mine, double2* __restrict__ peer, int l, int s, int b,
                uint64_t total) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t lbit = uint64_t(1) << l;
    uint64_t off[kIlp];
    double2 x[kIlp], y[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t j = first + uint64_t(i) * kThreads;
        if (j < total) {
            uint64_t o;
            if (s < 0) {
                o = insert0(j, l);
            } else {
                int lb = l < s ? l : s, hb = l < s ? s : l;
                o = insert0(insert0(j, lb), hb) | (uint64_t(b) << s);
            }
            o |= uint64_t(1 - b) << l;
            off[i] = o;
            x[i] = mine[o];
            y[i] = peer[o ^ lbit];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t j = first + uint64_t(i) * kThreads;
        if (j < total) {
            mine[off[i]] = y[i];
            peer[off[i] ^ lbit] = x[i];
        }
    }
}

// SWAP of two local qubits a < c (all states of the handle): amplitudes with
// (bit a, bit c) = (1, 0) trade places with (0, 1).
__global__ void __launch_bounds__(kThreads)
    k_swap_local(double2* __restrict__ psi, int m, int a, int c, uint64_t total) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t qmask = (uint64_t(1) << (m - 2)) - 1;
    uint64_t lo[kIlp];
    double2 x[kIlp], y[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total) {
            uint64_t st = p >> (m - 2), j = p & qmask;
            uint64_t o = insert0(insert0(j, a), c);
            lo[i] = (st << m) | o | (uint64_t(1) << a);
            x[i] = psi[lo[i]];
            y[i] = psi[lo[i] ^ (uint64_t(1) << a) ^ (uint64_t(1) << c)];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total) {
            psi[lo[i]] = y[i];
            psi[lo[i] ^ (uint64_t(1) << a) ^ (uint64_t(1) << c)] = x[i];
        }
    }
}

}  // namespace

void launch_swap_peer(double2* mine, double2* peer, int m, int l, int rank_bit, cudaStream_t st) {
    int s = -1;
    uint64_t total;
    if (m >= 2) {
        s = (l == m - 1) ? m - 2 : m - 1;
        total = uint64_t(1) << (m - 2);
    } else {
        if (rank_bit != 0) return;  // m == 1: the lower rank moves the single pair
        total = 1;
    }
    uint64_t per_block = kThreads * kIlp;
    unsigned grid = unsigned((total + per_block - 1) / per_block);
    k_swap_peer<<<grid ? grid : 1, kThreads, 0, st>>>(mine, peer, l, s, rank_bit, total);
}

void launch_swap_local(double2* psi, int m, int num_states, int a, int c, cudaStream_t st) {
    if (a > c) {
        int t = a;
        a = c;
        c = t;
    }
    uint64_t total = uint64_t(num_states) << (m - 2);
    uint64_t per_block = kThreads * kIlp;
    unsigned grid = unsigned((total + per_block - 1) / per_block);
    k_swap_local<<<grid ? grid : 1, kThreads, 0, st>>>(psi, m, a, c, total);
}

void launch_exchange_peer(double2* mine, double2* peer, int m, bool is_lower, const double* u_dev,
                          int control_local, cudaStream_t s) {
    int split_bit = m - 1;
    if (control_local == split_bit) split_bit = m - 2;
    uint64_t total;
    if (split_bit < 0) {
        if (!is_lower) return;
        total = (uint64_t(1) << m) >> (control_local >= 0 ? 1 : 0);
    } else {
        total = uint64_t(1) << (m - 1);
        if (control_local >= 0) total >>= 1;
    }
    uint64_t per_block = kThreads * kIlp;
    unsigned grid = unsigned((total + per_block - 1) / per_block);
    k_exchange_peer<<<grid ? grid : 1, kThreads, 0, s>>>(mine, peer, m, split_bit, is_lower ? 1 : 0,
                                                         control_local, total, u_dev);
}

void launch_pair_update_halves(double2* a, double2* b, uint64_t count, uint64_t first_offset,
                               const double* u_dev, int control_local, cudaStream_t s) {
    uint64_t g = (count + 255) / 256;
    if (g > 148ull * 16) g = 148ull * 16;
    k_pair_halves<<<unsigned(g ? g : 1), 256, 0, s>>>(a, b, count, first_offset, control_local,
                                                       u_dev);
}

}  // namespace qsb
