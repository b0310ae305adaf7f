// Gate kernels of the B200 state-vector core.
//
//  k_gate1q      one 2x2 gate on a local qubit: a streaming pass, 128-bit
//                double2 loads/stores, ILP pairs per thread
//                (reference: apply_local_one_qubit_gate, statevector.py:162-177)
//  k_controlled  control-mask compaction: thread j -> the j-th pair with control
//                bit 1, so only the control=1 half is read and written
//                (reference: apply_local_controlled_gate, statevector.py:180-195)
//  k_cut_phase   psi_i *= lut[cut(i)] (statevector.py:198-206 + graphs.py:35-42)
//  k_tile        fused pass: a 2^12-amplitude tile in shared memory, gates
//                applied in program order in register "rounds" of 4 qubits;
//                one HBM read + write for a whole run of gates.
#include "common.cuh"

namespace qsb {

namespace {

__device__ __forceinline__ void load_u(double2 u[4], const double* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = __ldg(q + k);
}

constexpr int kThreads = 256;
constexpr int kIlp = 4;

__global__ void __launch_bounds__(kThreads) k_gate1q(double2* __restrict__ psi, int m, int q,
                                                     uint64_t total_pairs,
                                                     const double* __restrict__ mats,
                                                     uint64_t offset, uint64_t stride) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t qmask = (uint64_t(1) << q) - 1;
    const uint64_t hmask = (uint64_t(1) << (m - 1)) - 1;
    const uint64_t step = uint64_t(1) << q;
    double2 u[4];
    if (stride == 0) load_u(u, mats + offset);
    uint64_t lo[kIlp];
    double2 a[kIlp], b[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            uint64_t s = p >> (m - 1), j = p & hmask;
            lo[i] = (s << m) | ((j & ~qmask) << 1) | (j & qmask);
            a[i] = psi[lo[i]];
            b[i] = psi[lo[i] + step];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            if (stride != 0) load_u(u, mats + offset + (p >> (m - 1)) * stride);
            pair_update(a[i], b[i], u);
            psi[lo[i]] = a[i];
            psi[lo[i] + step] = b[i];
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_controlled(double2* __restrict__ psi, int m, int c,
                                                         int t, uint64_t total_pairs,
                                                         const double* __restrict__ mats,
                                                         uint64_t offset, uint64_t stride,
                                                         int diag_one) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const int lowb = c < t ? c : t, highb = c < t ? t : c;
    const uint64_t qmask = (uint64_t(1) << (m - 2)) - 1;
    const uint64_t cbit = uint64_t(1) << c, tbit = uint64_t(1) << t;
    double2 u[4];
    if (stride == 0) load_u(u, mats + offset);
    uint64_t lo[kIlp];
    double2 a[kIlp], b[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            uint64_t s = p >> (m - 2), j = p & qmask;
            uint64_t x = insert0(insert0(j, lowb), highb) | cbit;
            lo[i] = (s << m) | x;
            if (!diag_one) a[i] = psi[lo[i]];
            b[i] = psi[lo[i] | tbit];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            if (stride != 0) load_u(u, mats + offset + (p >> (m - 2)) * stride);
            if (diag_one) {
                // u = diag(1, z): a is unchanged and b' = u11*b (the u10*a term is
                // a signed zero); only the control=1, target=1 quarter moves.
                psi[lo[i] | tbit] = cmul(u[3], b[i]);
            } else {
                pair_update(a[i], b[i], u);
                psi[lo[i]] = a[i];
                psi[lo[i] | tbit] = b[i];
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_cut_phase(double2* __restrict__ psi, int m,
                                                        uint64_t total, uint64_t rank_offset,
                                                        const __grid_constant__ CutTerms ct,
                                                        const double* __restrict__ mats,
                                                        uint64_t offset, uint64_t stride) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t lmask = (uint64_t(1) << m) - 1;
    double2 v[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t idx = first + uint64_t(i) * kThreads;
        if (idx < total) v[i] = psi[idx];
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t idx = first + uint64_t(i) * kThreads;
        if (idx < total) {
            uint64_t s = idx >> m;
            int k = cut_of(rank_offset | (idx & lmask), ct);
            const double2* lut = reinterpret_cast<const double2*>(mats + offset + s * stride);
            // reference: partition.amplitudes *= np.exp(-1j*angles): psi is the left operand
            psi[idx] = cmul(v[i], __ldg(lut + k));
        }
    }
}

// ---- fused tile pass ------------------------------------------------------------

constexpr int kTileAmps = 1 << kTileLog2;
constexpr int kRegAmps = 1 << kRegLog2;
constexpr int kLoadsPerThread = kTileAmps / kTileThreads;  // 16

// 2x2 update on register bit J of the 16 amplitudes a thread holds; with
// reg_control the pair is skipped unless register bit cval of its index is 1.
template <int J>
__device__ __forceinline__ void reg_gate(double2 (&a)[kRegAmps], const double2 u[4],
                                         bool reg_control, int cval) {
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) {
        if ((k >> J) & 1) continue;
        if (reg_control && !((k >> cval) & 1)) continue;
        pair_update(a[k], a[k | (1 << J)], u);
    }
}

__global__ void __launch_bounds__(kTileThreads, 2)
    k_tile(double2* __restrict__ psi, const TilePass* __restrict__ pass_dev,
           const double* __restrict__ mats, const __grid_constant__ CutTerms ct) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + sizeof(double2) * kTileAmps);
    TilePass* pass_s = reinterpret_cast<TilePass*>(smem_raw + sizeof(double2) * kTileAmps +
                                                   sizeof(uint64_t) * (kTileAmps >> 3));
    const int tid = threadIdx.x;
    {
        // the pass description (rounds, gates, shared matrices) is read once per
        // persistent CTA and then served from shared memory (uniform broadcasts)
        const uint4* src = reinterpret_cast<const uint4*>(pass_dev);
        uint4* dst = reinterpret_cast<uint4*>(pass_s);
        for (int i = tid; i < int(sizeof(TilePass) / 16); i += kTileThreads) dst[i] = src[i];
        __syncthreads();
    }
    const TilePass& P = *pass_s;
    const int low_run = P.low_run;
    const int nrows = kTileAmps >> low_run;
    const uint64_t lowmask = (uint64_t(1) << low_run) - 1;
    // row offsets: deposit of the row index into the tile bits above the low run
    for (int r = tid; r < nrows; r += kTileThreads) {
        uint64_t off = 0;
        for (int k = 0; k < kTileLog2 - low_run; ++k)
            if ((r >> k) & 1) off |= uint64_t(1) << P.tile_bits[low_run + k];
        rowoff[r] = off;
    }
    __syncthreads();

    const int m = P.m;
    const int tps_log2 = m - kTileLog2;
    for (uint64_t tile_id = blockIdx.x; tile_id < P.num_tiles; tile_id += gridDim.x) {
        const uint64_t s = tile_id >> tps_log2;
        uint64_t x = tile_id & (P.tiles_per_state - 1);
#pragma unroll
        for (int k = 0; k < kTileLog2; ++k) x = insert0(x, P.tile_bits[k]);
        const uint64_t base_local = x;                  // local offset of tile element 0
        double2* gbase = psi + ((s << m) | base_local);

        // HBM -> shared: consecutive threads read consecutive amplitudes of a row
#pragma unroll
        for (int h = 0; h < kLoadsPerThread; h += 8) {
            double2 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                int e = tid + (h + i) * kTileThreads;
                v[i] = gbase[rowoff[e >> low_run] + (e & lowmask)];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) tile[swz(tid + (h + i) * kTileThreads)] = v[i];
        }
        __syncthreads();

        for (int r = 0; r < P.num_rounds; ++r) {
            const Round& R = P.rounds[r];
            const int eb = R.dlo[tid & 15] | R.dhi[tid >> 4];
            const int sb = R.slo[tid & 15] ^ R.shi[tid >> 4];
            double2 a[kRegAmps];
#pragma unroll
            for (int k = 0; k < kRegAmps; ++k) a[k] = tile[sb ^ R.sk[k]];

            const int g_end = R.first_gate + R.num_gates;
            for (int g = R.first_gate; g < g_end; ++g) {
                const TileGate& G = P.gates[g];
                if (G.kind == QS_KIND_CUTPHASE) {
                    const double2* lut =
                        reinterpret_cast<const double2*>(mats + G.offset + s * G.stride);
#pragma unroll
                    for (int k = 0; k < kRegAmps; ++k) {
                        const int e = eb | R.dk[k];
                        uint64_t local = base_local + rowoff[e >> low_run] + (uint64_t(e) & lowmask);
                        a[k] = cmul(a[k], __ldg(lut + cut_of(P.rank_offset | local, ct)));
                    }
                    continue;
                }
                if (G.ctype == 2 && !((eb >> G.cval) & 1)) continue;
                if (G.ctype == 3 && !((base_local >> G.cval) & 1)) continue;
                double2 u[4];
                if (G.stride == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) u[q] = make_double2(G.u[2 * q], G.u[2 * q + 1]);
                } else {
                    load_u(u, mats + G.offset + s * G.stride);
                }
                const bool rc = G.ctype == 1;
                switch (G.j) {
                    case 0: reg_gate<0>(a, u, rc, G.cval); break;
                    case 1: reg_gate<1>(a, u, rc, G.cval); break;
                    case 2: reg_gate<2>(a, u, rc, G.cval); break;
                    default: reg_gate<3>(a, u, rc, G.cval); break;
                }
            }
#pragma unroll
            for (int k = 0; k < kRegAmps; ++k) tile[sb ^ R.sk[k]] = a[k];
            __syncthreads();
        }

        // shared -> HBM
#pragma unroll
        for (int i = 0; i < kLoadsPerThread; ++i) {
            int e = tid + i * kTileThreads;
            gbase[rowoff[e >> low_run] + (e & lowmask)] = tile[swz(e)];
        }
        __syncthreads();
    }
}

__global__ void k_fill(double2* __restrict__ psi, uint64_t count, double2 value) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        psi[i] = value;
}

__global__ void k_scale(double2* __restrict__ psi, uint64_t count, double f) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double2 v = psi[i];
        psi[i] = make_double2(__dmul_rn(v.x, f), __dmul_rn(v.y, f));
    }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Box-Muller on two 53-bit uniforms derived from (seed, state, global index):
// the same amplitude gets the same value for any rank split.
__global__ void k_gaussian(double2* __restrict__ psi, uint64_t per_state, int m, uint64_t total,
                           uint64_t rank_offset, uint64_t seed) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t s = i >> m, g = rank_offset | (i & (per_state - 1));
        uint64_t h = splitmix(seed ^ splitmix(s * 0x632BE59BD9B4E019ull ^ splitmix(g)));
        uint64_t h2 = splitmix(h);
        double u1 = (double((h >> 11) + 1)) * 0x1.0p-53;  // (0, 1]
        double u2 = double(h2 >> 11) * 0x1.0p-53;         // [0, 1)
        double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        psi[i] = make_double2(r * cs, r * sn);
    }
}

inline unsigned grid_for(uint64_t work, uint64_t per_block) {
    uint64_t g = (work + per_block - 1) / per_block;
    return unsigned(g == 0 ? 1 : g);
}

inline unsigned stream_grid(uint64_t count) {
    // grid-stride loops: a few waves over the 148 SMs
    uint64_t g = (count + 255) / 256;
    uint64_t cap = 148ull * 16;
    return unsigned(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void launch_gate1q(double2* psi, int m, int num_states, int q, const double* mats, uint64_t offset,
                   uint64_t stride, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << (m - 1);
    k_gate1q<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(psi, m, q, total, mats, offset,
                                                                    stride);
}

void launch_controlled(double2* psi, int m, int num_states, int c, int t, const double* mats,
                       uint64_t offset, uint64_t stride, bool diag_one, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << (m - 2);
    k_controlled<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(
        psi, m, c, t, total, mats, offset, stride, diag_one ? 1 : 0);
}

void launch_cut_phase(double2* psi, int m, int num_states, uint64_t rank_offset, const CutTerms& ct,
                      const double* mats, uint64_t offset, uint64_t stride, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << m;
    k_cut_phase<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(psi, m, total, rank_offset,
                                                                       ct, mats, offset, stride);
}

size_t tile_smem_bytes() {
    return sizeof(double2) * kTileAmps + sizeof(uint64_t) * (kTileAmps >> 3) + sizeof(TilePass);
}

void launch_tile_pass(double2* psi, const TilePass& pass, const TilePass* pass_dev,
                      const double* mats, const CutTerms& ct, cudaStream_t s) {
    static bool configured = false;
    const size_t smem = tile_smem_bytes();
    static int sms = 148, per_sm = 2;
    if (!configured) {
        cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile, kTileThreads, smem);
        if (per_sm < 1) per_sm = 1;
        configured = true;
    }
    uint64_t grid = uint64_t(sms) * per_sm;
    if (grid > pass.num_tiles) grid = pass.num_tiles;
    k_tile<<<unsigned(grid), kTileThreads, smem, s>>>(psi, pass_dev, mats, ct);
}

void launch_fill(double2* psi, uint64_t count, double2 value, cudaStream_t s) {
    k_fill<<<stream_grid(count), 256, 0, s>>>(psi, count, value);
}

void launch_scale(double2* psi, uint64_t count, double factor, cudaStream_t s) {
    k_scale<<<stream_grid(count), 256, 0, s>>>(psi, count, factor);
}

void launch_gaussian(double2* psi, uint64_t per_state, int num_states, uint64_t rank_offset,
                     uint64_t seed, cudaStream_t s) {
    int m = 0;
    while ((uint64_t(1) << m) < per_state) ++m;
    uint64_t total = per_state * uint64_t(num_states);
    k_gaussian<<<stream_grid(total), 256, 0, s>>>(psi, per_state, m, total, rank_offset, seed);
}

}  // namespace qsb
