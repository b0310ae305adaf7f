// Factored programs (QS_FUSE_FACTORED): the same operator as the user's gate
// list with about a quarter of the FP64 work per fused pass.
//
// Every uncontrolled 1q gate with a shared unitary matrix U is written
//     U = k * diag(1, za) * R * diag(1, zb),   R = [[c,-s],[s,c]],  c,s >= 0,
// and R as a shear times a scalar: c*[[1,-t],[t,1]] with t = s/c.  A shear pair
// update is 4 FMAs (2 FP64 instructions per amplitude) against numpy's 10 per
// amplitude for a general complex 2x2 (statevector.py:144-150).  A large t
// costs no accuracy (fma(-t, y, x) rounds once, relative to |x - t y|, and the
// scale c brings the result back), only growth: the amplitudes grow by at most
// 1/c per shear until the scalar is applied, so gates with c < 1e-9 stay exact
// and a scalar pass is inserted when the pending scale passes 2^-600.  The
// rest is bookkeeping that costs nothing per amplitude:
//  * scalars commute with everything: k and the shear scale multiply into one
//    constant applied once at the end;
//  * diag(1, z) on qubit q commutes with every gate that does not mix q
//    (gates on other qubits, controls on q, cut phases, diagonal gates), so
//    the za of one gate on q and the zb of the next gate on q meet and merge
//    into one pre-diagonal of that shear (complex multiply of its b member);
//  * the zb of the FIRST mixing gate on q moves to the program start and the
//    za of the LAST one to the program end, where the diagonals of all qubits
//    form one product diagonal D(i) = prod_q z_q^{bit_q(i)} (kKindDiagN),
//    evaluated per tile from byte tables plus a walk over the register bits.
// For a layer of 1q gates on distinct qubits (BASELINE config 2's sweep, the
// 1q layers of configs 1 and 4) this leaves one shear per gate plus D_in and
// D_out.  Controlled gates, per-state matrix tables, non-unitary matrices and
// cut phases stay exact.  Errors are a few ulps per gate (the tests bound them
// by the north_star 1e-12 on amplitudes).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>

#include "common.cuh"

namespace qsb {

namespace {
using cd = std::complex<double>;

cd unit(cd z) { return z / std::abs(z); }

// K * (re + i im) without libgcc's IEEE-special-case complex multiply
// (__muldc3), and max(|Re|, |Im|) for the rescale trigger instead of a hypot:
// the per-state loops of a 512-state QAOA program (80 gates x 512 states)
// run 1.1 ms -> less on the host
inline cd scale_by(cd k, double re, double im) {
    return cd(k.real() * re - k.imag() * im, k.real() * im + k.imag() * re);
}
inline double mag_bound(cd k) { return std::max(std::fabs(k.real()), std::fabs(k.imag())); }

cd entry(const double* u, int i) { return cd(u[2 * i], u[2 * i + 1]); }

bool is_unitary(const cd u[4]) {
    // U^dagger U == I to 1e-12
    const cd g00 = std::conj(u[0]) * u[0] + std::conj(u[2]) * u[2];
    const cd g11 = std::conj(u[1]) * u[1] + std::conj(u[3]) * u[3];
    const cd g01 = std::conj(u[0]) * u[1] + std::conj(u[2]) * u[3];
    return std::abs(g00 - 1.0) <= 1e-12 && std::abs(g11 - 1.0) <= 1e-12 && std::abs(g01) <= 1e-12;
}
}  // namespace

bool decompose_2x2(const double* m, double out[10]) {
    cd u[4];
    for (int i = 0; i < 4; ++i) u[i] = entry(m, i);
    for (int i = 0; i < 8; ++i)
        if (!std::isfinite(m[i])) return false;
    if (u[1] == 0.0 && u[2] == 0.0) return false;  // diagonal: merged as a diagonal instead
    if (!is_unitary(u)) return false;
    const double a00 = std::abs(u[0]), a01 = std::abs(u[1]), a10 = std::abs(u[2]),
                 a11 = std::abs(u[3]);
    double c = std::sqrt(0.5 * (a00 * a00 + a11 * a11));
    double s = std::sqrt(0.5 * (a01 * a01 + a10 * a10));
    const double r = std::hypot(c, s);
    c /= r;
    s /= r;
    // u00 = k c, u01 = -k s zb, u10 = k za s, u11 = k za zb c.  The phases come
    // from the two large entries, the ratio (or product) from the two small
    // ones, so an error in a small entry's phase only moves small entries.
    cd k, za, zb;
    int form;
    double t, scale;
    if (c >= s) {
        k = unit(u[0]);
        const cd P = unit(u[3]) / k;                                         // za * zb
        const cd Q = (a01 > 0 && a10 > 0) ? -unit(u[2]) * std::conj(unit(u[1])) : cd(1.0);  // za / zb
        za = std::sqrt(P * Q);
        zb = P / za;
        if (std::real(std::conj(k * za) * u[2]) < 0) za = -za, zb = -zb;  // u10 = +k za s
    } else {
        const cd Q = -unit(u[2]) * std::conj(unit(u[1]));                          // za / zb
        const cd P = (a00 > 0 && a11 > 0) ? unit(u[3]) * std::conj(unit(u[0])) : cd(1.0);  // za * zb
        za = std::sqrt(P * Q);
        zb = P / za;
        k = unit(u[2]) / za;  // u10 = k za s
        if (a00 > 0 && std::real(std::conj(k) * u[0]) < 0) za = -za, zb = -zb, k = -k;  // u00 = +k c
    }
    if (c < 1e-9) return false;  // nearly anti-diagonal: t would exceed 1e9
    form = 0;
    t = s / c;
    scale = c;
    za = unit(za);
    zb = unit(zb);
    out[0] = k.real(), out[1] = k.imag();
    out[2] = za.real(), out[3] = za.imag();
    out[4] = zb.real(), out[5] = zb.imag();
    out[6] = form, out[7] = t, out[8] = scale, out[9] = 0;
    return true;
}

void factor_program(const qs_gate* gates, int count, const double* mats, uint64_t mats_len, int m,
                    int num_states, int num_edges, uint64_t phase_support, FactoredProgram* out,
                    bool batch_flush) {
    out->gates.clear();
    out->extra.clear();
    out->factored = 0;
    std::vector<cd> pending(m, cd(1.0)), din(m, cd(1.0));
    std::vector<char> mixed(m, 0);
    cd K(1.0);
    const int ntab = (m + 7) / 8;

    auto params = [&](const double* p8) {
        const uint64_t off = mats_len + out->extra.size();
        out->extra.insert(out->extra.end(), p8, p8 + 8);
        return off;
    };
    auto emit = [&](int kind, int target, uint64_t off) {
        qs_gate g;
        memset(&g, 0, sizeof(g));
        g.kind = kind;
        g.target = target;
        g.control = -1;
        g.offset = off;
        g.stride = 0;
        out->gates.push_back(g);
    };
    // product diagonal sum over set bits: byte tables with `scalar` in table 0
    auto diag_tables = [&](const std::vector<cd>& z, cd scalar) {
        while (out->extra.size() % 2) out->extra.push_back(0.0);  // 16-byte aligned entries
        const uint64_t off = mats_len + out->extra.size();
        std::vector<cd> T(size_t(ntab) * 256);
        for (int c = 0; c < ntab; ++c) {
            cd* t = T.data() + c * 256;
            t[0] = 1.0;
            for (int v = 1; v < 256; ++v) {
                const int b = __builtin_ctz(v), q = 8 * c + b;
                t[v] = t[v & (v - 1)] * (q < m ? z[q] : cd(1.0));
            }
        }
        for (int v = 0; v < 256; ++v) T[v] *= scalar;
        for (const cd& x : T) out->extra.push_back(x.real()), out->extra.push_back(x.imag());
        for (int q = 0; q < 64; ++q) {
            const cd x = q < m ? z[q] : cd(1.0);
            out->extra.push_back(x.real()), out->extra.push_back(x.imag());
        }
        qs_gate g;
        memset(&g, 0, sizeof(g));
        g.kind = kKindDiagN;
        g.target = -1;
        g.control = -1;
        g.reserved = ntab;
        g.offset = off;
        return g;
    };
    auto diag1 = [&](int q, cd z) {
        const double p[8] = {0, 0, 0, 0, z.real(), z.imag(), 0, 0};
        emit(kKindDiag1, q, params(p));
    };
    // per-state pending diagonals (pool gates whose diagonals differ between
    // states, e.g. noise trajectories): psp[q][s] replaces pending[q] (then 1)
    std::vector<std::vector<cd>> psp(m);
    auto per_state_rows = [&](int kind, int q, const std::vector<double>& t, const std::vector<cd>& z,
                              bool has_z) {
        while (out->extra.size() % 2) out->extra.push_back(0.0);
        const uint64_t off = mats_len + out->extra.size();
        for (int st = 0; st < num_states; ++st) {
            const double p[8] = {t.empty() ? 0.0 : t[st], 0, has_z ? 1.0 : 0.0, 0,
                                 z[st].real(), z[st].imag(), 0, 0};
            out->extra.insert(out->extra.end(), p, p + 8);
        }
        qs_gate g;
        memset(&g, 0, sizeof(g));
        g.kind = kind;
        g.target = q;
        g.control = -1;
        g.offset = off;
        g.stride = 8;
        g.reserved = 1;  // per-state pre-diagonals: not for the lean kernel's shared pre
        out->gates.push_back(g);
    };
    auto flush = [&](int q) {  // make the pending diagonal on q explicit before a mixing gate
        if (!psp[q].empty()) {
            per_state_rows(kKindDiag1, q, {}, psp[q], true);
            psp[q].clear();
        }
        if (pending[q] != 1.0) {
            if (!mixed[q]) din[q] *= pending[q];
            else diag1(q, pending[q]);
            pending[q] = 1.0;
        }
    };
    // a gate's matrix entries: the caller's table, or the extra entries (merged gates)
    auto mat = [&](const qs_gate& g, int st) -> const double* {
        const uint64_t off = g.offset + uint64_t(st) * g.stride;
        return off >= mats_len ? out->extra.data() + (off - mats_len) : mats + off;
    };
    auto diagonal_for_all_states = [&](const qs_gate& g) {
        for (int s = 0; s < num_states; ++s) {
            const double* u = mat(g, s);
            if (u[2] != 0 || u[3] != 0 || u[4] != 0 || u[5] != 0) return false;
            if (g.stride == 0) break;
        }
        return true;
    };

    // per-state scalars (pool mode): k * scale of the per-state shears
    std::vector<cd> Ks(num_states, cd(1.0));
    bool per_state_k = false;
    auto per_state_scalars = [&]() {
        while (out->extra.size() % 2) out->extra.push_back(0.0);
        const uint64_t off = mats_len + out->extra.size();
        for (int s = 0; s < num_states; ++s) {
            const double p[8] = {Ks[s].real(), Ks[s].imag(), 0, 0, 0, 0, 0, 0};
            out->extra.insert(out->extra.end(), p, p + 8);
            Ks[s] = 1.0;
        }
        qs_gate g;
        memset(&g, 0, sizeof(g));
        g.kind = kKindScalar;
        g.target = -1;
        g.control = -1;
        g.offset = off;
        g.stride = 8;
        out->gates.push_back(g);
    };
    std::vector<double> fs;
    // the 20 mixers of a QAOA layer share one per-state table (GateQueue keys):
    // its factorisation is computed once, and the shear rows are emitted once
    // per (table, pre-diagonal)
    uint64_t fs_off = ~uint64_t(0), fs_stride = 0;
    bool fs_same = true;
    struct RowKey { uint64_t off, stride, at; bool has_pre; cd pre; };
    std::vector<RowKey> row_cache;
    auto per_state_shear = [&](const qs_gate& g) {
        const int q = g.target;
        fs.resize(size_t(num_states) * 10);
        bool same = true;
        const bool cached = g.offset == fs_off && g.stride == fs_stride && g.offset < mats_len;
        if (cached) same = fs_same;
        for (int st = 0; st < num_states && !cached; ++st) {
            double* f = fs.data() + 10 * st;
            const double* u = mat(g, st);
            // RX(theta) = [[c, -is], [-is, c]] = c * diag(1, i) [[1,-t],[t,1]] diag(1, -i)
            // with t = -s/c: closed form (the QAOA mixer, 80 x 512 matrices a step)
            if (u[0] == u[6] && u[1] == 0 && u[7] == 0 && u[2] == 0 && u[4] == 0 && u[3] == u[5] &&
                std::abs(u[0] * u[0] + u[3] * u[3] - 1.0) <= 1e-12 && std::abs(u[0]) >= 1e-9) {
                f[0] = u[0] < 0 ? -1.0 : 1.0, f[1] = 0.0;
                f[2] = 0.0, f[3] = 1.0, f[4] = 0.0, f[5] = -1.0;
                f[6] = 0.0, f[7] = u[3] / u[0], f[8] = std::abs(u[0]), f[9] = 0.0;
            } else if (!decompose_2x2(u, f)) {
                fs_off = ~uint64_t(0);  // fs is partly overwritten
                return false;
            }
            if (st == 0 && (f[3] < 0 || (f[3] == 0 && f[2] < 0))) {
                // canonical sign (Im za >= 0): consecutive gates of one family
                // (RX layers) then meet with za * zb = 1 and need no pre-diagonal
                f[2] = -f[2], f[3] = -f[3], f[4] = -f[4], f[5] = -f[5], f[7] = -f[7];
            }
            // the same diagonals for every state; (za, zb) and (-za, -zb) are
            // the same factorisation with the sign of t flipped
            const cd za0(fs[2], fs[3]), zb0(fs[4], fs[5]), za1(f[2], f[3]), zb1(f[4], f[5]);
            if (std::abs(za1 - za0) <= 1e-13 && std::abs(zb1 - zb0) <= 1e-13) continue;
            if (std::abs(za1 + za0) <= 1e-13 && std::abs(zb1 + zb0) <= 1e-13) {
                // keep the state's triple consistent (the per-state path uses it)
                f[2] = -f[2], f[3] = -f[3], f[4] = -f[4], f[5] = -f[5], f[7] = -f[7];
                continue;
            }
            same = false;
        }
        fs_off = g.offset, fs_stride = g.stride, fs_same = same;
        if (!same || !psp[q].empty()) {
            // per-state diagonals: every state's pre-diagonal and pending za
            // are its own (no product diagonal at the program ends)
            std::vector<double> t(num_states);
            std::vector<cd> pre(num_states), za_s(num_states);
            bool any_pre = false;
            double small = 1.0;
            for (int st = 0; st < num_states; ++st) {
                const double* f = fs.data() + 10 * st;
                const cd zb(f[4], f[5]);
                pre[st] = (psp[q].empty() ? pending[q] : psp[q][st]) * zb;
                any_pre |= pre[st] != 1.0;
                za_s[st] = cd(f[2], f[3]);
                t[st] = f[7];
                Ks[st] = scale_by(Ks[st], f[0] * f[8], f[1] * f[8]);
                small = std::min(small, mag_bound(Ks[st]));
            }
            per_state_rows(kKindShear, q, t, pre, any_pre);
            out->factored++;
            per_state_k = true;
            pending[q] = 1.0;
            psp[q] = za_s;
            mixed[q] = 1;
            if (small < 0x1p-600) per_state_scalars();
            return true;
        }
        const cd za(fs[2], fs[3]), zb(fs[4], fs[5]);
        const cd pre = pending[q] * zb;
        bool has_pre = false;
        if (!mixed[q]) din[q] *= pre;
        else has_pre = pre != 1.0;
        uint64_t off = ~uint64_t(0);
        if (g.offset < mats_len)
            for (const RowKey& k : row_cache)
                if (k.off == g.offset && k.stride == g.stride && k.has_pre == has_pre &&
                    (!has_pre || k.pre == pre))
                    off = k.at;
        const bool emit = off == ~uint64_t(0);
        if (emit) {
            while (out->extra.size() % 2) out->extra.push_back(0.0);
            off = mats_len + out->extra.size();
            if (g.offset < mats_len) row_cache.push_back({g.offset, g.stride, off, has_pre, pre});
            out->extra.reserve(out->extra.size() + size_t(num_states) * 8);
        }
        double small = 1.0;
        for (int st = 0; st < num_states; ++st) {
            const double* f = fs.data() + 10 * st;
            if (emit) {
                // z is (1, 0) without a pre-diagonal: lean pool passes read it per state
                const double p[8] = {f[7], 0, has_pre ? 1.0 : 0.0, 0, has_pre ? pre.real() : 1.0,
                                     has_pre ? pre.imag() : 0.0, 0, 0};
                out->extra.insert(out->extra.end(), p, p + 8);
            }
            Ks[st] = scale_by(Ks[st], f[0] * f[8], f[1] * f[8]);
            small = std::min(small, mag_bound(Ks[st]));
        }
        qs_gate s8;
        memset(&s8, 0, sizeof(s8));
        s8.kind = kKindShear;
        s8.target = q;
        s8.control = -1;
        s8.offset = off;
        s8.stride = 8;
        out->gates.push_back(s8);
        out->factored++;
        per_state_k = true;
        pending[q] = za;
        mixed[q] = 1;
        if (small < 0x1p-600) per_state_scalars();
        return true;
    };

    // Gate fusion first: consecutive 1q gates on one qubit (nothing else on that
    // qubit in between) become one matrix -- U2*U1, per state when either is --
    // emitted where the qubit is next touched (or at the end).  A noise
    // trajectory's rotation after each mixer RX then costs one shear, not two.
    std::vector<qs_gate> prog;
    {
        struct Acc {
            qs_gate g;
            int n = 0;                    // original gates merged
            std::vector<cd> m;            // 4 entries per state (1 state when shared)
        };
        std::vector<Acc> acc(m);
        // last gate of `prog` that touches each qubit: consecutive controlled
        // gates on one (control, target) pair fuse like 1q gates do
        std::vector<int> last_touch(m, -1);
        auto touch = [&](const qs_gate& g) {
            const int at = int(prog.size());
            if (g.kind == QS_KIND_CUTPHASE) {
                for (int q = 0; q < m; ++q)
                    if ((phase_support >> q) & 1) last_touch[q] = at;
                return;
            }
            last_touch[g.target] = at;
            if (g.kind == QS_KIND_CTRL) last_touch[g.control] = at;
        };
        auto load = [&](const qs_gate& g, std::vector<cd>& dst) {
            const int ns = g.stride ? num_states : 1;
            dst.resize(4 * size_t(ns));
            for (int st = 0; st < ns; ++st) {
                const uint64_t off = g.offset + uint64_t(st) * g.stride;
                const double* u = off >= mats_len ? out->extra.data() + (off - mats_len) : mats + off;
                for (int e = 0; e < 4; ++e) dst[4 * st + e] = cd(u[2 * e], u[2 * e + 1]);
            }
        };
        auto emit_acc = [&](int q) {
            Acc& a = acc[q];
            if (a.n == 0) return;
            if (a.n == 1) {
                touch(a.g);
                prog.push_back(a.g);
            } else {
                const int ns = int(a.m.size() / 4);
                while (out->extra.size() % 2) out->extra.push_back(0.0);
                qs_gate g = a.g;
                g.offset = mats_len + out->extra.size();
                g.stride = ns > 1 ? 8 : 0;
                for (const cd& x : a.m) out->extra.push_back(x.real()), out->extra.push_back(x.imag());
                touch(g);
                prog.push_back(g);
                out->factored += a.n - 1;  // the merged-away gates cost nothing
            }
            a.n = 0;
            a.m.clear();
        };
        std::vector<cd> u2;
        for (int i = 0; i < count; ++i) {
            const qs_gate& g = gates[i];
            if (g.kind == QS_KIND_1Q) {
                Acc& a = acc[g.target];
                if (a.n == 0) {
                    a.g = g;
                    load(g, a.m);
                } else {
                    load(g, u2);
                    const int n1 = int(a.m.size() / 4), n2 = int(u2.size() / 4);
                    const int ns = std::max(n1, n2);
                    std::vector<cd> r(4 * size_t(ns));
                    for (int st = 0; st < ns; ++st) {
                        const cd* x = u2.data() + 4 * (n2 > 1 ? st : 0);    // later gate
                        const cd* y = a.m.data() + 4 * (n1 > 1 ? st : 0);   // earlier gate
                        r[4 * st + 0] = x[0] * y[0] + x[1] * y[2];
                        r[4 * st + 1] = x[0] * y[1] + x[1] * y[3];
                        r[4 * st + 2] = x[2] * y[0] + x[3] * y[2];
                        r[4 * st + 3] = x[2] * y[1] + x[3] * y[3];
                    }
                    a.m.swap(r);
                }
                a.n++;
                continue;
            }
            if (g.kind == QS_KIND_CTRL) {
                // batch_flush: the 1q gates of every qubit the run of controlled
                // gates touches come before its first gate, so that their
                // pending diagonals can leave as ONE product diagonal
                // (and every other accumulated gate: left behind, a qubit the run
                // does not touch would get a pass of its own after the run)
                if (batch_flush) {
                    for (int q = 0; q < m; ++q) emit_acc(q);
                } else {
                    emit_acc(g.target);
                    emit_acc(g.control);
                }
                // the previous gate on both qubits is a controlled gate on the same
                // pair: one controlled gate with the product matrix (config 3's
                // CNOT, CPhase, controlled-U on a pair become one gate)
                const int li = last_touch[g.control];
                if (li >= 0 && li == last_touch[g.target] && prog[li].kind == QS_KIND_CTRL &&
                    prog[li].control == g.control && prog[li].target == g.target) {
                    std::vector<cd> y, x;
                    load(prog[li], y);  // earlier gate
                    load(g, x);         // later gate
                    const int n1 = int(y.size() / 4), n2 = int(x.size() / 4);
                    const int ns = std::max(n1, n2);
                    while (out->extra.size() % 2) out->extra.push_back(0.0);
                    const uint64_t off = mats_len + out->extra.size();
                    for (int st = 0; st < ns; ++st) {
                        const cd* b = x.data() + 4 * (n2 > 1 ? st : 0);
                        const cd* a = y.data() + 4 * (n1 > 1 ? st : 0);
                        const cd r[4] = {b[0] * a[0] + b[1] * a[2], b[0] * a[1] + b[1] * a[3],
                                         b[2] * a[0] + b[3] * a[2], b[2] * a[1] + b[3] * a[3]};
                        for (const cd& v : r) out->extra.push_back(v.real()), out->extra.push_back(v.imag());
                    }
                    prog[li].offset = off;
                    prog[li].stride = ns > 1 ? 8 : 0;
                    out->factored++;  // the merged-away gate costs nothing
                    continue;
                }
            } else {  // cut phase: every vertex of the graph
                for (int q = 0; q < m; ++q)
                    if ((phase_support >> q) & 1) emit_acc(q);
            }
            touch(g);
            prog.push_back(g);
        }
        for (int q = 0; q < m; ++q) emit_acc(q);
    }
    for (size_t i = 0; i < prog.size(); ++i) {
        const qs_gate g = prog[i];
        if (g.kind == QS_KIND_CUTPHASE) {  // diagonal: commutes with every pending diagonal
            out->gates.push_back(g);
            continue;
        }
        const int q = g.target;
        if (g.kind == QS_KIND_CTRL) {
            if (!diagonal_for_all_states(g)) {
                if (batch_flush) {
                    // the pending diagonals of every target this run of controlled
                    // gates mixes: one product diagonal (a lean op, 2 complex
                    // products per amplitude) instead of a Diag1 per target on k_tile
                    std::vector<int> ts;
                    for (size_t j = i; j < prog.size() && prog[j].kind == QS_KIND_CTRL; ++j) {
                        const int t = prog[j].target;
                        if (diagonal_for_all_states(prog[j]) || !psp[t].empty() || !mixed[t] ||
                            pending[t] == 1.0 || std::find(ts.begin(), ts.end(), t) != ts.end())
                            continue;
                        ts.push_back(t);
                    }
                    if (ts.size() >= 4) {
                        // ... and with them every other pending diagonal and the
                        // scalar: nothing is left for a D_out behind the run
                        std::vector<cd> z(m, cd(1.0));
                        for (int t = 0; t < m; ++t)
                            if (psp[t].empty() && mixed[t] && pending[t] != 1.0)
                                z[t] = pending[t], pending[t] = 1.0;
                        out->gates.push_back(diag_tables(z, K));
                        K = 1.0;
                    }
                }
                flush(q);
                mixed[q] = 1;
            }
            out->gates.push_back(g);
            continue;
        }
        // QS_KIND_1Q
        if (g.stride != 0 && diagonal_for_all_states(g)) {
            // per-state diagonal gate (per-state RZ(gamma_s), pure-dephasing
            // noise, fused products that come out diagonal): u_s = u00_s *
            // diag(1, u11_s / u00_s) -- the scalar joins the per-state scalars,
            // the diagonal the per-state pending diagonal of q (it commutes with
            // everything pending there).  Non-unitary diagonals run exact.
            bool unit_all = true;
            for (int st = 0; st < num_states && unit_all; ++st) {
                const double* u = mat(g, st);
                unit_all = std::abs(std::abs(entry(u, 0)) - 1.0) <= 1e-12 &&
                           std::abs(std::abs(entry(u, 3)) - 1.0) <= 1e-12;
            }
            if (!unit_all) {
                out->gates.push_back(g);  // diagonal: no flush needed
                continue;
            }
            std::vector<cd> z(num_states);
            for (int st = 0; st < num_states; ++st) {
                const double* u = mat(g, st);
                const cd u00 = entry(u, 0), u11 = entry(u, 3);
                z[st] = (psp[q].empty() ? pending[q] : psp[q][st]) * (u11 / u00);
                Ks[st] *= u00;
            }
            psp[q].swap(z);
            pending[q] = 1.0;
            per_state_k = true;
            out->factored++;
            continue;
        }
        if (g.stride != 0) {
            // per-state matrices (pool mode): a per-state shear when every
            // state's matrix factors with the same diagonals (e.g. the QAOA
            // mixer RX(2 beta_s): za = -i, zb = i for every beta), the scales
            // and k going to per-state scalars
            if (!diagonal_for_all_states(g) && !per_state_shear(g)) {
                flush(q);
                mixed[q] = 1;
                out->gates.push_back(g);
            }
            continue;
        }
        const double* u = mat(g, 0);
        const cd u00 = entry(u, 0), u11 = entry(u, 3);
        if (entry(u, 1) == 0.0 && entry(u, 2) == 0.0 && std::abs(std::abs(u00) - 1.0) <= 1e-12 &&
            std::abs(std::abs(u11) - 1.0) <= 1e-12) {
            K *= u00;  // diag(u00, u11) = u00 * diag(1, u11/u00)
            if (psp[q].empty()) pending[q] *= u11 / u00;
            else for (cd& z : psp[q]) z *= u11 / u00;
            out->factored++;  // absorbed: costs nothing per amplitude
            continue;
        }
        double f[10];
        if (!decompose_2x2(u, f)) {
            flush(q);
            mixed[q] = 1;
            out->gates.push_back(g);
            continue;
        }
        const cd k(f[0], f[1]), za(f[2], f[3]), zb(f[4], f[5]);
        if (!psp[q].empty()) {
            // shared gate after per-state diagonals on q: per-state pre-diagonals
            std::vector<cd> pre(num_states);
            for (int st = 0; st < num_states; ++st) pre[st] = psp[q][st] * zb;
            per_state_rows(kKindShear, q, std::vector<double>(num_states, f[7]), pre, true);
            K *= k * f[8];
            out->factored++;
            psp[q].clear();
            pending[q] = za;
            mixed[q] = 1;
            continue;
        }
        const cd pre = pending[q] * zb;
        K *= k * f[8];
        bool has_pre = false;
        if (!mixed[q]) din[q] *= pre;
        else has_pre = pre != 1.0;
        const double p[8] = {f[7], f[6], has_pre ? 1.0 : 0.0, 0, has_pre ? pre.real() : 1.0,
                             has_pre ? pre.imag() : 0.0, 0, 0};
        emit(kKindShear, q, params(p));
        out->factored++;
        pending[q] = za;
        mixed[q] = 1;
        // the amplitudes grow by 1/c per shear; a scalar pass keeps them far
        // from overflow in long programs
        if (std::abs(K) < 0x1p-600) {
            out->gates.push_back(diag_tables(std::vector<cd>(m, cd(1.0)), K));
            K = 1.0;
        }
    }
    bool any_in = false;
    for (int q = 0; q < m; ++q) any_in |= din[q] != 1.0;
    if (any_in) out->gates.insert(out->gates.begin(), diag_tables(din, cd(1.0)));
    bool any_out = K != 1.0;
    for (int q = 0; q < m; ++q) any_out |= pending[q] != 1.0;
    if (any_out) out->gates.push_back(diag_tables(pending, K));
    for (int q = 0; q < m; ++q)  // per-state pending diagonals close the program
        if (!psp[q].empty()) per_state_rows(kKindDiag1, q, {}, psp[q], true);
    // padding row of the lean pool passes: t = 0, z = (1, 0)
    while (out->extra.size() % 2) out->extra.push_back(0.0);
    out->zero_off = mats_len + out->extra.size();
    {
        const double pad[8] = {0, 0, 0, 0, 1, 0, 0, 0};
        out->extra.insert(out->extra.end(), pad, pad + 8);
    }
    if (per_state_k) {
        // the per-state scalars ride on a cut phase when the program has one
        // (each state's LUT row times its scalar: no extra pass op)
        int cut = -1;
        for (int i = int(out->gates.size()) - 1; i >= 0 && cut < 0; --i)
            if (out->gates[i].kind == QS_KIND_CUTPHASE) cut = i;
        if (cut < 0) {
            per_state_scalars();
        } else {
            qs_gate& g = out->gates[cut];
            const uint64_t len = 2 * uint64_t(num_edges + 1);
            const double* src = g.offset >= mats_len ? out->extra.data() + (g.offset - mats_len)
                                                     : mats + g.offset;
            std::vector<double> rows(len * num_states);
            for (int st = 0; st < num_states; ++st)
                for (uint64_t e = 0; e < len; e += 2) {
                    const double* x = src + uint64_t(st) * g.stride + e;
                    const cd v = cd(x[0], x[1]) * Ks[st];
                    rows[st * len + e] = v.real(), rows[st * len + e + 1] = v.imag();
                }
            while (out->extra.size() % 2) out->extra.push_back(0.0);
            g.offset = mats_len + out->extra.size();
            g.stride = len;
            out->extra.insert(out->extra.end(), rows.begin(), rows.end());
        }
    }
}

// ---- commutation-aware order (factored programs only) -----------------------
// Gates that commute may run in either order; in the factored mode (results to
// the 1e-12 tolerance, not bit-identical) the program is re-ordered so that the
// greedy pass planner packs more gates into each tile pass.  Two gates commute
// unless one MIXES a qubit (target of a non-diagonal matrix) that the other
// touches at all; diagonal actions (controls, diagonal matrices, cut phases,
// product diagonals) commute with each other.  The list schedule keeps every
// dependency and fills a pass first with ready gates that need no new tile bit,
// then with ready gates in program order while the tile has room.  A QAOA layer
// pair [RX(0..11), cut, RX(0..11)] then shares one pass: the config-5 pool
// circuit needs 6 passes instead of 10.
void schedule_program(std::vector<qs_gate>& gates, int m, uint64_t phase_support,
                      const double* mats, int num_states, bool lean_first) {
    const int n = int(gates.size());
    if (n < 3) return;
    const uint64_t all = m >= 64 ? ~uint64_t(0) : (uint64_t(1) << m) - 1;
    std::vector<uint64_t> mix(n, 0), dia(n, 0);
    auto diagonal = [&](const qs_gate& g) {
        for (int st = 0; st < num_states; ++st) {
            const double* u = mats + g.offset + uint64_t(st) * g.stride;
            if (u[2] != 0 || u[3] != 0 || u[4] != 0 || u[5] != 0) return false;
            if (g.stride == 0) break;
        }
        return true;
    };
    for (int i = 0; i < n; ++i) {
        const qs_gate& g = gates[i];
        const uint64_t t = g.target >= 0 ? uint64_t(1) << g.target : 0;
        switch (g.kind) {
            case QS_KIND_CUTPHASE: dia[i] = phase_support; break;
            case kKindDiagN: dia[i] = all; break;
            // a mid-program rescale must stay between the shears around it
            // (pulled forward, the product of several would underflow)
            case kKindScalar: dia[i] = all; break;
            case kKindDiag1: dia[i] = t; break;
            case kKindShear: mix[i] = t; break;
            case QS_KIND_CTRL:
                dia[i] = uint64_t(1) << g.control;
                (diagonal(g) ? dia[i] : mix[i]) |= t;
                break;
            default: (diagonal(g) ? dia[i] : mix[i]) |= t; break;
        }
    }
    std::vector<std::vector<int>> succ(n);
    std::vector<int> npred(n, 0);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i)
            if ((mix[i] & (mix[j] | dia[j])) || (dia[i] & mix[j])) {
                succ[i].push_back(j);
                ++npred[j];
            }
    std::vector<int> ready;  // kept sorted by program index
    for (int i = 0; i < n; ++i)
        if (npred[i] == 0) ready.push_back(i);
    std::vector<qs_gate> out;
    out.reserve(n);
    const uint64_t low = m >= kTileLog2 ? kLowMask : 0;
    while (!ready.empty()) {
        uint64_t need = low, round_set = 0;
        int rounds = 1, count = 0, diags = 0;
        int pass_class = 0;  // max class of the pass's gates (gate_class)
        for (;;) {
            int pick = -1;
            uint64_t pick_need = 0, pick_rs = 0;
            int pick_nr = 0;
            // lean_first: a pass opens with a lean gate when one is ready (else a
            // CNOT, else anything), a pass of lean gates takes no other kind and
            // a pass of CNOTs only CNOTs (config 4: the Haar layer stays on the
            // lean kernels, the CNOT passes run as permutations on k_perm)
            int open_class = 2;
            if (lean_first && count == 0)
                for (int gi : ready) open_class = std::min(open_class, gate_class(gates[gi], mats));
            // preference: no new register round and no new tile bit, then no
            // new tile bit, then program order
            for (int tier = 0; tier < 3 && pick < 0; ++tier) {
                for (size_t k = 0; k < ready.size(); ++k) {
                    const qs_gate& g = gates[ready[k]];
                    if (lean_first) {
                        const int cls = gate_class(g, mats);
                        if (count == 0 && cls != open_class) continue;
                        if (count > 0 && pass_class < 2 && cls != pass_class) continue;
                        if (count > 0 && pass_class == 2 && cls == 0 && tier == 2) continue;
                    }
                    uint64_t nn = need, rs = round_set;
                    int nr = rounds;
                    if (kind_has_target(g.kind)) {
                        const uint64_t b = uint64_t(1) << g.target;
                        if (tier < 2 && !(need & b)) continue;
                        nn |= b;
                        if (!(rs & b)) {
                            if (__builtin_popcountll(rs) >= kRegLog2) {
                                if (tier == 0) continue;
                                rs = 0;
                                ++nr;
                            }
                            rs |= b;
                        }
                    }
                    if (count > 0 && (__builtin_popcountll(nn) > kTileLog2 || nr > kMaxRounds ||
                                      count + 1 > kMaxPassGates ||
                                      (g.kind == kKindDiagN && diags >= kMaxPassDiags)))
                        continue;
                    pick = int(k);
                    pick_need = nn, pick_rs = rs, pick_nr = nr;
                    break;
                }
            }
            if (pick < 0) break;
            const int gi = ready[pick];
            ready.erase(ready.begin() + pick);
            out.push_back(gates[gi]);
            need = pick_need, round_set = pick_rs, rounds = pick_nr;
            ++count;
            pass_class = std::max(pass_class, gate_class(gates[gi], mats));
            diags += gates[gi].kind == kKindDiagN;
            for (int j : succ[gi])
                if (--npred[j] == 0) ready.insert(std::lower_bound(ready.begin(), ready.end(), j), j);
        }
    }
    gates.swap(out);
}

}  // namespace qsb
