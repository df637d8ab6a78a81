// Diagnostics: cycles per row of a record-solve round on independent chains
// (one per lane; x[i] depends on x[i-1] of the same chain through shared
// memory), with the pieces of the production round switched on and off.
// Build + run on a GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/round_bench.cu -o /tmp/rb && /tmp/rb
#include <cstdio>
#include <cstdint>

constexpr unsigned long long kSent = 0xFFFFFFFFFFFFFFFFull;
constexpr int N = 512;  // rows per chain
constexpr int kLanes = 32;

__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u64(uint32_t a, unsigned long long v) {
    asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void lds_f64x2(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void lds_s32x2(uint32_t a, int& x, int& y) {
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}

struct Rec {  // as TrsvRec
    double v[4];
    double d, y;
    short idx[4];
    int pad[2];
};

constexpr int F_VOTE = 1;      // converged rounds: while (__any_sync) { if (!ready) continue; ... }
constexpr int F_RING = 2;      // records staged by cp.async (ring of 4), next row read from the ring + adopt
constexpr int F_FOUR = 4;      // four operand loads + four sentinel tests + four products
constexpr int F_DIVCHK = 8;    // exponent test, __ddiv_rn fallback branch
constexpr int F_STG = 16;      // st.relaxed.gpu of x
constexpr int F_REGCHAIN = 32; // chain operand forwarded in a register (no smem read for it)
constexpr int F_NOZERO = 64;   // t = br - sp with a zero select instead of acc = 0 + sp
constexpr int F_SOA = 128;     // ring laid out [slot][16-byte chunk][lane] (no bank conflicts)
constexpr int F_WINSKEW = 256; // window rows of lane l start at a bank-skewed offset

template <int F>
__global__ void chain(const Rec* rec, const double* b, double* x, long long* cycles, int slot) {
    extern __shared__ __align__(16) unsigned long long smem[];
    // layout: zero word, window [kLanes][N], ring [kLanes][4][10]
    const int lane = threadIdx.x;
    unsigned long long* zero = smem;
    unsigned long long* win = smem + 2;
    unsigned long long* ring = win + kLanes * N;
    for (int i = lane; i < kLanes * N; i += 32) win[i] = kSent;
    if (lane == 0) zero[0] = 0;
    __syncwarp();
    const uint32_t zero_a = static_cast<uint32_t>(__cvta_generic_to_shared(zero));
    const uint32_t win_a = static_cast<uint32_t>(__cvta_generic_to_shared(win)) + 8u * lane * (N - ((F & F_WINSKEW) ? 4 : 0));
    const uint32_t ring_base = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
    const uint32_t ring_a = ring_base + 320u * lane;
    // chunk c (16 bytes) of slot k
    auto rc = [&](int k, int c) -> uint32_t {
        return (F & F_SOA) ? ring_base + 16u * ((k * 5 + c) * kLanes + lane) : ring_a + 80u * k + 16u * c;
    };
    const Rec* myrec = rec + lane * N;
    const double* myb = b + lane * N;
    double* myx = x + lane * N;
    // current row state
    int r = 0, st = 0;
    double v0 = 0, v1 = 0, v2 = 0, v3 = 0, d = 0, y = 0, br = 0;
    uint32_t a0 = zero_a, a1 = zero_a, a2 = zero_a, a3 = zero_a;
    double xprev = 0.0;
    auto stage = [&](int k) {
        const int s = st < N ? st : 0;
        const char* src = reinterpret_cast<const char*>(myrec + s);
        cpa16(rc(k, 0), src); cpa16(rc(k, 1), src + 16); cpa16(rc(k, 2), src + 32); cpa16(rc(k, 3), src + 48);
        cpa8(rc(k, 4), myb + s);
        asm volatile("st.shared.s32 [%0], %1;" ::"r"(rc(k, 4) + 8), "r"(st < N ? st : -1) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        ++st;
    };
    auto from_ring = [&](int k) {
        int rr, pad, m01, m23;
        double br2, dd;
        lds_s32x2(rc(k, 4) + 8, rr, pad);
        lds_f64x2(rc(k, 0), v0, v1);
        lds_f64x2(rc(k, 1), v2, v3);
        lds_f64x2(rc(k, 2), d, y);
        lds_s32x2(rc(k, 3), m01, m23);
        lds_f64x2(rc(k, 4), br2, dd);
        br = br2;
        r = rr;
        // operand addresses: the chain operand (row r-1 of this lane) in slot 3
        a3 = win_a + 8u * (r - 1);
        a0 = a1 = a2 = zero_a + 0u * static_cast<uint32_t>(m01 + m23);
        if (r == 0) a3 = zero_a;
    };
    if (F & F_RING) {
        for (int k = 0; k < 4; ++k) stage(k);
        asm volatile("cp.async.wait_group 3;" ::: "memory");
        from_ring(0);
        stage(0);
    } else {
        v0 = v1 = v2 = 0.0;
        v3 = -0.5;
        d = 2.0;
        y = 0.5;
        br = 1.0;
        a3 = zero_a;
    }
    int h = 1;
    long long t0 = clock64();
    auto body = [&]() -> bool {  // returns false when not ready
        unsigned long long u0 = 0, u1 = 0, u2 = 0, u3;
        if (F & F_FOUR) {
            u0 = lds_u64(a0);
            u1 = lds_u64(a1);
            u2 = lds_u64(a2);
        }
        if (F & F_REGCHAIN) {
            u3 = static_cast<unsigned long long>(__double_as_longlong(xprev));
        } else {
            u3 = lds_u64(a3);
        }
        if ((F & F_FOUR) ? (u0 == kSent || u1 == kSent || u2 == kSent || u3 == kSent) : (u3 == kSent)) return false;
        int nr = r + 1;
        if (F & F_RING) asm volatile("cp.async.wait_group 3;" ::: "memory");
        double sp;
        if (F & F_FOUR) {
            sp = __dmul_rn(v0, __longlong_as_double(static_cast<long long>(u0)));
            sp = __dadd_rn(sp, __dmul_rn(v1, __longlong_as_double(static_cast<long long>(u1))));
            sp = __dadd_rn(sp, __dmul_rn(v2, __longlong_as_double(static_cast<long long>(u2))));
            sp = __dadd_rn(sp, __dmul_rn(v3, __longlong_as_double(static_cast<long long>(u3))));
        } else {
            sp = __dmul_rn(v3, __longlong_as_double(static_cast<long long>(u3)));
        }
        double t;
        if (F & F_NOZERO) {
            const double t1 = __dsub_rn(br, sp);
            t = (static_cast<unsigned long long>(__double_as_longlong(sp)) << 1) == 0 ? br : t1;
        } else {
            const double acc = __dadd_rn(0.0, sp);
            t = __dsub_rn(br, acc);
        }
        double xr;
        const double q0 = __dmul_rn(t, y);
        const double rq = __fma_rn(-d, q0, t);
        xr = __fma_rn(y, rq, q0);
        if (F & F_DIVCHK) {
            const unsigned en = (static_cast<unsigned>(__double2hiint(t)) >> 20) & 0x7FFu;
            const unsigned ed = (static_cast<unsigned>(__double2hiint(d)) >> 20) & 0x7FFu;
            if (!(en - 523u <= 1000u && ed - 523u <= 1000u)) xr = __ddiv_rn(t, d);
            if (static_cast<unsigned long long>(__double_as_longlong(xr)) == kSent) xr = __longlong_as_double(0x7FF8000000000000ll);
        }
        sts_u64(win_a + 8u * r, static_cast<unsigned long long>(__double_as_longlong(xr)));
        if (F & F_STG) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(myx + r), "l"(__double_as_longlong(xr)) : "memory");
        xprev = xr;
        if (F & F_RING) {
            from_ring(h);
            stage(h);
            h = (h + 1) & 3;
        } else {
            r = nr;
            a3 = win_a + 8u * (r - 1);
        }
        return true;
    };
    if (F & F_VOTE) {
        while (__any_sync(0xFFFFFFFFu, r >= 0 && r < N)) {
            if (!(r >= 0 && r < N)) continue;
            body();
        }
    } else {
        while (r >= 0 && r < N) body();
    }
    long long t1 = clock64();
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == slot) cycles[0] = t1 - t0;
    myx[N - 1] += xprev * 1e-300;
}


// The production record loop (sptrsv_rec_kernel, converged rounds) on the
// same chains, SoA ring; G_* flags change its schedule.
constexpr int G_EARLYSTAGE = 1;  // restage the ring slot right after reading it (before the FP chain)
constexpr int G_NODIV = 2;       // no exponent test / __ddiv_rn fallback
constexpr int G_NOSTG = 4;       // no st.relaxed.gpu of x
constexpr int G_PRED = 8;        // readiness predicates the body instead of `continue`
constexpr int G_RING8 = 16;      // ring of 8
template <int G>
__global__ void chain2(const Rec* rec, const double* b, double* x, long long* cycles, int slot) {
    extern __shared__ __align__(16) unsigned long long smem[];
    constexpr int kR = (G & G_RING8) ? 8 : 4;
    const int lane = threadIdx.x;
    const int kT = blockDim.x;
    unsigned long long* zero = smem;
    unsigned long long* win = smem + 2;
    unsigned long long* ring = win + kLanes * N;
    for (int i = lane; i < kLanes * N; i += 32) win[i] = kSent;
    if (lane == 0) zero[0] = 0;
    __syncwarp();
    const uint32_t zero_a = static_cast<uint32_t>(__cvta_generic_to_shared(zero));
    const uint32_t win_a = static_cast<uint32_t>(__cvta_generic_to_shared(win)) + 8u * lane * (N - 4);
    const uint32_t ring_base = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
    auto ch = [&](int k, int c) -> uint32_t { return ring_base + 16u * static_cast<uint32_t>((k * 5 + c) * kT + lane); };
    const Rec* myrec = rec + lane * N;
    const double* myb = b + lane * N;
    double* myx = x + lane * N;
    int st = 0;
    auto stage = [&](int k) {
        const int s = st < N ? st : 0;
        const char* src = reinterpret_cast<const char*>(myrec + s);
        if (st < N) {
            cpa16(ch(k, 0), src); cpa16(ch(k, 1), src + 16); cpa16(ch(k, 2), src + 32); cpa16(ch(k, 3), src + 48);
            cpa8(ch(k, 4), myb + s);
        }
        asm volatile("st.shared.s32 [%0], %1;" ::"r"(ch(k, 4) + 8), "r"(st < N ? st : -1) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        ++st;
    };
    struct Raw { int r, pad, m01, m23; double v0, v1, v2, v3, d, y, br, dd; };
    auto load_raw = [&](Raw& w, int k) {
        lds_s32x2(ch(k, 4) + 8, w.r, w.pad);
        lds_f64x2(ch(k, 0), w.v0, w.v1);
        lds_f64x2(ch(k, 1), w.v2, w.v3);
        lds_f64x2(ch(k, 2), w.d, w.y);
        lds_s32x2(ch(k, 3), w.m01, w.m23);
        lds_f64x2(ch(k, 4), w.br, w.dd);
    };
    int r; uint32_t a0, a1, a2, a3; double v0, v1, v2, v3, d, y, br;
    auto adopt = [&](const Raw& w) {
        r = w.r; v0 = w.v0; v1 = w.v1; v2 = w.v2; v3 = w.v3; d = w.d; y = w.y; br = w.br;
        a0 = zero_a + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(w.m01 & 0xFFFF)) + 1);
        a1 = zero_a + 8u * static_cast<uint32_t>((w.m01 >> 16) + 1);
        a2 = zero_a + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(w.m23 & 0xFFFF)) + 1);
        a3 = r > 0 ? win_a + 8u * (r - 1) : zero_a;
    };
    for (int k = 0; k < kR; ++k) stage(k);
    asm volatile("cp.async.wait_group %0;" ::"n"(kR - 1) : "memory");
    { Raw w; load_raw(w, 0); adopt(w); }
    stage(0);
    int h = 1;
    double xlast = 0;
    long long t0 = clock64();
    while (__any_sync(0xFFFFFFFFu, r >= 0)) {
        if (!(G & G_PRED) && r < 0) continue;
        const unsigned long long u0 = lds_u64(a0), u1 = lds_u64(a1), u2 = lds_u64(a2), u3 = lds_u64(a3);
        const bool ready = r >= 0 && u0 != kSent && u1 != kSent && u2 != kSent && u3 != kSent;
        if (!(G & G_PRED) && !ready) continue;
        asm volatile("cp.async.wait_group %0;" ::"n"(kR - 1) : "memory");
        Raw w;
        load_raw(w, h);
        if ((G & G_EARLYSTAGE) && ready) stage(h);
        double sp = __dmul_rn(v0, __longlong_as_double(static_cast<long long>(u0)));
        sp = __dadd_rn(sp, __dmul_rn(v1, __longlong_as_double(static_cast<long long>(u1))));
        sp = __dadd_rn(sp, __dmul_rn(v2, __longlong_as_double(static_cast<long long>(u2))));
        sp = __dadd_rn(sp, __dmul_rn(v3, __longlong_as_double(static_cast<long long>(u3))));
        const double acc = __dadd_rn(0.0, sp);
        const double t = __dsub_rn(br, acc);
        const double q0 = __dmul_rn(t, y);
        const double rq = __fma_rn(-d, q0, t);
        double xr = __fma_rn(y, rq, q0);
        if (!(G & G_NODIV)) {
            const unsigned en = (static_cast<unsigned>(__double2hiint(t)) >> 20) & 0x7FFu;
            const unsigned ed = (static_cast<unsigned>(__double2hiint(d)) >> 20) & 0x7FFu;
            if (!(en - 523u <= 1000u && ed - 523u <= 1000u)) xr = __ddiv_rn(t, d);
            if (static_cast<unsigned long long>(__double_as_longlong(xr)) == kSent) xr = __longlong_as_double(0x7FF8000000000000ll);
        }
        if (!(G & G_PRED) || ready) {
            sts_u64(win_a + 8u * r, static_cast<unsigned long long>(__double_as_longlong(xr)));
            if (!(G & G_NOSTG))
                asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(myx + r), "l"(__double_as_longlong(xr)) : "memory");
            xlast = xr;
            adopt(w);
            if (!(G & G_EARLYSTAGE)) stage(h);
            h = (h + 1) & (kR - 1);
        }
    }
    long long t1 = clock64();
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == slot) cycles[0] = t1 - t0;
    myx[N - 1] += xlast * 1e-300;
}

template <int G>
void run2(const char* name, const Rec* rec, const double* b, double* x, long long* cyc, int lanes) {
    const size_t smem = (2 + kLanes * N + kLanes * 8 * 10) * 8;
    cudaFuncSetAttribute(chain2<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
        chain2<G><<<1, lanes, smem>>>(rec, b, x, cyc, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-52s lanes %2d  %7.1f cycles/row\n", name, lanes, double(h) / N);
}

template <int F>
void run(const char* name, const Rec* rec, const double* b, double* x, long long* cyc, int lanes) {
    const size_t smem = (2 + kLanes * N + kLanes * 40) * 8;
    cudaFuncSetAttribute(chain<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
        chain<F><<<1, lanes, smem>>>(rec, b, x, cyc, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-52s lanes %2d  %7.1f cycles/row\n", name, lanes, double(h) / N);
}

int main() {
    Rec* rec;
    double *b, *x;
    long long* cyc;
    const int n = kLanes * N;
    cudaMalloc(&rec, n * sizeof(Rec));
    cudaMalloc(&b, n * 8);
    cudaMalloc(&x, n * 8);
    cudaMalloc(&cyc, 64);
    Rec* hr = new Rec[n];
    double* hb = new double[n];
    for (int i = 0; i < n; ++i) {
        hr[i] = Rec{{0.0, 0.0, 0.0, -0.5}, 2.0, 0.5, {-1, -1, -1, 0}, {0, 0}};
        hb[i] = 1.0 + (i % 97) * 1e-3;
    }
    cudaMemcpy(rec, hr, n * sizeof(Rec), cudaMemcpyHostToDevice);
    cudaMemcpy(b, hb, n * 8, cudaMemcpyHostToDevice);
    for (int lanes : {1, 32}) {
        run2<0>("PROD order", rec, b, x, cyc, lanes);
        run2<G_EARLYSTAGE>("PROD early stage", rec, b, x, cyc, lanes);
        run2<G_NODIV>("PROD no div check", rec, b, x, cyc, lanes);
        run2<G_NOSTG>("PROD no STG", rec, b, x, cyc, lanes);
        run2<G_PRED>("PROD predicated", rec, b, x, cyc, lanes);
        run2<G_RING8>("PROD ring 8", rec, b, x, cyc, lanes);
        run2<G_NODIV | G_NOSTG>("PROD no div, no STG", rec, b, x, cyc, lanes);
        run2<G_EARLYSTAGE | G_NODIV>("PROD early stage, no div", rec, b, x, cyc, lanes);
    }
    for (int lanes : {1, 32}) {
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_RING | F_SOA>("all, SoA ring", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_RING | F_SOA | F_WINSKEW>("all, SoA ring, skewed window", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_SOA | F_WINSKEW>("all but ring, skewed window", rec, b, x, cyc, lanes);
        run<F_WINSKEW>("minimal, skewed window", rec, b, x, cyc, lanes);
        run<F_RING | F_SOA | F_WINSKEW>("+SoA ring, skewed window", rec, b, x, cyc, lanes);
        run<0>("minimal", rec, b, x, cyc, lanes);
        run<F_REGCHAIN>("minimal, chain in register", rec, b, x, cyc, lanes);
        run<F_VOTE>("+vote loop", rec, b, x, cyc, lanes);
        run<F_FOUR>("+four operands", rec, b, x, cyc, lanes);
        run<F_DIVCHK>("+division check", rec, b, x, cyc, lanes);
        run<F_STG>("+STG", rec, b, x, cyc, lanes);
        run<F_RING>("+ring", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_RING>("all (production-like)", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_RING | F_NOZERO>("all, zero select", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG | F_RING | F_REGCHAIN>("all, chain in register", rec, b, x, cyc, lanes);
        run<F_FOUR | F_DIVCHK | F_STG | F_RING>("all but vote", rec, b, x, cyc, lanes);
        run<F_VOTE | F_DIVCHK | F_STG | F_RING>("all but four", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_STG | F_RING>("all but division check", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_RING>("all but STG", rec, b, x, cyc, lanes);
        run<F_VOTE | F_FOUR | F_DIVCHK | F_STG>("all but ring", rec, b, x, cyc, lanes);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
