// splinerecon.cu — C ABI (include/splinerecon.h) over the sm_100a reconstruction kernels.
//
// Replaces the reference's batch evaluator PlanInterpreter.eval_batch -> _eval_batch
// (runtime.py:244-248, :363-408).  sp_plan_create is the analogue of
// PlanInterpreter.__init__ + _batch_tables (runtime.py:219-230, :256-272): it validates the
// flattened EvaluationPlan, derives the site reach (halo) and picks the kernel family:
//   * tensor-product B-spline (separable closed form, caller-asserted + verified here),
//   * a plan-specialised kernel generated at build time (codegen.py) and matched by the
//     plan's exact canonical content,
//   * the generic table-driven kernel.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/splinerecon.h"
#include "sp_common.cuh"
#include "sp_evaluators.cuh"
#include "sp_launch.cuh"
#include "sp_tma.cuh"
#include "sp_bcc_linear.cuh"


// generated plan kernels + kGenerated[] registry (codegen.py)
#include "generated/registry.inc"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define SP_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) return fail(SP_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

// Class record packing shared with the generated kernels (codegen.py: decode_class()).
//   x: kernel | perm_i << (4+2i) | (sign_i<0) << (10+i) | rho_i << (13+2i) | (tau_i<0) << (19+i)
//   y: (t_i + 128) << 8i          z: (pib_i/d + 128) << 8i
struct HostClass {
    int kernel;
    int perm[3], sign[3], t[3], rho[3], tau[3], pibd[3];
};

bool signed_perm(const double* m, int perm[3], int sign[3]) {
    int used = 0;
    for (int i = 0; i < 3; ++i) {
        int nz = 0;
        for (int j = 0; j < 3; ++j) {
            const double v = m[3 * i + j];
            if (v == 0.0) continue;
            if (v != 1.0 && v != -1.0) return false;
            ++nz;
            perm[i] = j;
            sign[i] = v > 0 ? 1 : -1;
        }
        if (nz != 1) return false;
        used |= 1 << perm[i];
    }
    return used == 7;
}

}  // namespace

namespace sp {
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace sp

struct sp_plan {
    sp_kernel_kind kind = SP_KIND_GENERIC;
    std::string name;
    int s = 3, M = 1;
    int diag[3] = {1, 1, 1};
    int shifts[SP_MAX_COSETS][3] = {};
    int reach_lo[3] = {0, 0, 0}, reach_hi[3] = {0, 0, 0};
    int tp_degree = -1;
    int N = 0;
    const sp::GenEntry* gen = nullptr;
    void* d_tables = nullptr;  // generated: sigma + class records; generic: GenericTables
    int table_bytes = 0;       // bytes staged into smem (generated only)
    std::vector<void*> allocs;
    int occ_f32 = 0, occ_f64 = 0;
    int num_sms = 148;
    bool bcc_tet = false;  // bcc_linear_rd: closed-form evaluator (sp_bcc_linear.cuh)
};

namespace {

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <typename V>
int upload(sp_plan* p, const std::vector<V>& v, const V** out) {
    void* d = nullptr;
    const size_t bytes = std::max<size_t>(v.size() * sizeof(V), 16);
    SP_CUDA(cudaMalloc(&d, bytes));
    p->allocs.push_back(d);
    if (!v.empty()) SP_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
    *out = reinterpret_cast<const V*>(d);
    return SP_OK;
}

uint64_t as_u64(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
}

// Canonical content of a plan: the exact sequence codegen.py:canonical_words() emits.
std::vector<uint64_t> canonical_words(const sp_plan_desc& d, int n_sites, int n_terms) {
    std::vector<uint64_t> w;
    auto I = [&](int64_t v) { w.push_back((uint64_t)v); };
    auto D = [&](double v) { w.push_back(as_u64(v)); };
    const int s = d.s;
    I(s); I(d.M);
    for (int i = 0; i < s; ++i) I(d.diag[i]);
    for (int k = 0; k < d.M; ++k)
        for (int i = 0; i < s; ++i) I(d.shifts[k][i]);
    I(d.Q);
    for (int j = 0; j < d.Q * s; ++j) I(d.normals[j]);
    for (int j = 0; j < d.Q; ++j) D(d.offsets[j]);
    I(d.r);
    for (int j = 0; j < d.r; ++j) I(d.sigma[j]);
    I(d.N);
    for (int c = 0; c < d.N; ++c) I(d.cls_kernel[c]);
    for (int j = 0; j < d.N * s * s; ++j) D(d.cls_T[j]);
    for (int j = 0; j < d.N * s; ++j) D(d.cls_t[j]);
    for (int j = 0; j < d.N * s * s; ++j) I(d.cls_piA[j]);
    for (int j = 0; j < d.N * s; ++j) I(d.cls_pib[j]);
    I(d.K);
    for (int j = 0; j <= d.K; ++j) I(d.kernel_group_start[j]);
    I(d.n_groups);
    for (int g = 0; g < d.n_groups; ++g) I(d.group_nspan[g]);
    for (int j = 0; j < d.n_groups * SP_MAX_DIM; ++j) I(d.group_span[j]);
    for (int j = 0; j <= d.n_groups; ++j) I(d.group_site_start[j]);
    for (int j = 0; j < n_sites * s; ++j) I(d.sites[j]);
    for (int j = 0; j <= d.n_groups; ++j) I(d.group_poly_start[j]);
    I(d.n_polys);
    for (int j = 0; j <= d.n_polys; ++j) I(d.poly_term_start[j]);
    for (int j = 0; j < n_terms * s; ++j) I(d.term_exps[j]);
    for (int j = 0; j < n_terms; ++j) D(d.term_coeffs[j]);
    return w;
}

double poly_eval_host(const sp_plan_desc& d, int p, const double y[3]) {
    double acc = 0.0;
    for (int t = d.poly_term_start[p]; t < d.poly_term_start[p + 1]; ++t) {
        double m = d.term_coeffs[t];
        for (int i = 0; i < 3; ++i) m *= std::pow(y[i], d.term_exps[3 * t + i]);
        acc += m;
    }
    return acc;
}

double bspline_w(int deg, int a, double t) {
    // weight of site floor(x) - deg + a; matches sp_evaluators.cuh BWeights
    const double s = 1.0 - t;
    switch (deg) {
        case 1: return a == 0 ? s : t;
        case 2: return a == 0 ? 0.5 * s * s : (a == 2 ? 0.5 * t * t : t * s + 0.5);
        case 3:
            if (a == 0) return s * s * s / 6.0;
            if (a == 3) return t * t * t / 6.0;
            if (a == 1) return (3 * t * t * t - 6 * t * t + 4) / 6.0;
            return (3 * s * s * s - 6 * s * s + 4) / 6.0;
    }
    return NAN;
}

// Numerical check of the caller's tensor-product assertion: plan weights (reconstructed
// from g and t_nums exactly as plancompile.py:676-699 lowers them) vs the closed form.
int verify_tensor(const sp_plan_desc& d, int deg) {
    if (deg < 1 || deg > 3) return fail(SP_ERR_UNSUPPORTED, "tensor-product degree %d not implemented", deg);
    if (d.M != 1 || d.Q != 0 || d.N != 1 || d.K != 1 || d.diag[0] != 1 || d.diag[1] != 1 || d.diag[2] != 1)
        return fail(SP_ERR_INVALID, "tp_degree asserted for a plan that is not single-coset Cartesian");
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            if (d.cls_T[3 * i + j] != (i == j ? 1.0 : 0.0) || d.cls_piA[3 * i + j] != (i == j ? 1 : 0))
                return fail(SP_ERR_INVALID, "tp_degree asserted for a plan with a non-identity class");
        }
    for (int i = 0; i < 3; ++i)
        if (d.cls_t[i] != 0.0 || d.cls_pib[i] != 0) return fail(SP_ERR_INVALID, "tp_degree: non-zero class shift");
    uint64_t st = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        return (double)(st >> 11) * (1.0 / 9007199254740992.0);
    };
    const int want = (deg + 1) * (deg + 1) * (deg + 1);
    for (int trial = 0; trial < 16; ++trial) {
        const double y[3] = {rnd(), rnd(), rnd()};
        std::vector<double> w(want, 0.0);
        int seen = 0;
        for (int g = d.kernel_group_start[0]; g < d.kernel_group_start[1]; ++g) {
            const int ns = d.group_nspan[g];
            const int p0 = d.group_poly_start[g];
            const double gv = poly_eval_host(d, p0, y);
            double t[3] = {0, 0, 0};
            for (int j = 0; j < ns; ++j) t[j] = gv == 0 ? 0.5 : poly_eval_host(d, p0 + 1 + j, y) / gv;
            for (int c = 0; c < (1 << ns); ++c) {
                const int* site = d.sites + 3 * (d.group_site_start[g] + c);
                double wc = gv;
                for (int j = 0; j < ns; ++j) wc *= ((c >> j) & 1) ? t[j] : 1.0 - t[j];
                int idx = 0;
                for (int i = 0; i < 3; ++i) {
                    const int a = site[i] + deg;
                    if (a < 0 || a > deg) return fail(SP_ERR_INVALID, "tp_degree: site outside the B-spline footprint");
                    idx = idx * (deg + 1) + a;
                }
                w[idx] += wc;
                ++seen;
            }
        }
        if (seen != want) return fail(SP_ERR_INVALID, "tp_degree: plan has %d sites, expected %d", seen, want);
        for (int a0 = 0; a0 <= deg; ++a0)
            for (int a1 = 0; a1 <= deg; ++a1)
                for (int a2 = 0; a2 <= deg; ++a2) {
                    const double ref = bspline_w(deg, a0, y[0]) * bspline_w(deg, a1, y[1]) * bspline_w(deg, a2, y[2]);
                    const double got = w[(a0 * (deg + 1) + a1) * (deg + 1) + a2];
                    if (std::fabs(ref - got) > 1e-9) return fail(SP_ERR_INVALID, "tp_degree: weights differ (%g vs %g)", got, ref);
                }
    }
    return SP_OK;
}

}  // namespace

extern "C" {

const char* sp_last_error(void) { return g_err.c_str(); }
const char* sp_version(void) { return "splinerecon 0.1.0 (sm_100a)"; }

int sp_plan_create(const sp_plan_desc* desc, sp_plan** out) {
    if (!desc || !out) return fail(SP_ERR_INVALID, "null argument");
    *out = nullptr;
    const sp_plan_desc& d = *desc;
    if (d.s != 3) return fail(SP_ERR_UNSUPPORTED, "only s == 3 plans are implemented on the GPU (got s=%d)", d.s);
    if (d.M < 1 || d.M > SP_MAX_COSETS) return fail(SP_ERR_UNSUPPORTED, "M=%d cosets not supported", d.M);
    if (d.Q < 0 || d.Q > 62) return fail(SP_ERR_UNSUPPORTED, "Q=%d planes not supported", d.Q);
    if (d.r < 1 || d.N < 1 || d.K < 1 || d.n_groups < 0 || d.n_polys < 0) return fail(SP_ERR_INVALID, "bad plan sizes");
    for (int i = 0; i < 3; ++i)
        if (d.diag[i] <= 0) return fail(SP_ERR_INVALID, "diag must be positive");
    for (int j = 0; j < d.r; ++j)
        if (d.sigma[j] < -1 || d.sigma[j] >= d.N) return fail(SP_ERR_INVALID, "sigma entry out of range");
    for (int c = 0; c < d.N; ++c)
        if (d.cls_kernel[c] < 0 || d.cls_kernel[c] >= d.K) return fail(SP_ERR_INVALID, "class kernel out of range");
    if (d.kernel_group_start[0] != 0 || d.kernel_group_start[d.K] != d.n_groups)
        return fail(SP_ERR_INVALID, "kernel_group_start inconsistent");
    for (int g = 0; g < d.n_groups; ++g) {
        const int ns = d.group_nspan[g];
        if (ns < 0 || ns > 3) return fail(SP_ERR_INVALID, "group span must be 0..3");
        if (d.group_site_start[g + 1] - d.group_site_start[g] != (1 << ns))
            return fail(SP_ERR_INVALID, "group %d: size != 2^len(span_axes)", g);
        if (d.group_poly_start[g + 1] - d.group_poly_start[g] != 1 + ns)
            return fail(SP_ERR_INVALID, "group %d: need g + one t_num per span axis", g);
    }
    const int n_sites = d.group_site_start[d.n_groups];
    if (d.group_poly_start[d.n_groups] != d.n_polys) return fail(SP_ERR_INVALID, "poly count inconsistent");
    const int n_terms = d.poly_term_start[d.n_polys];

    sp_plan* p = new sp_plan();
    p->s = d.s;
    p->M = d.M;
    p->N = d.N;
    for (int i = 0; i < 3; ++i) p->diag[i] = d.diag[i];
    for (int k = 0; k < d.M; ++k)
        for (int i = 0; i < 3; ++i) p->shifts[k][i] = d.shifts[k][i];

    // site offsets per class: (piA site + pib) / d must be integral (SURVEY.md §9 probe11)
    std::vector<int> site_off((size_t)d.N * n_sites * 3);
    bool first = true;
    for (int c = 0; c < d.N; ++c) {
        for (int g = 0; g < d.n_groups; ++g) {
            int kern = 0;
            while (d.kernel_group_start[kern + 1] <= g) ++kern;
            for (int sidx = d.group_site_start[g]; sidx < d.group_site_start[g + 1]; ++sidx) {
                for (int i = 0; i < 3; ++i) {
                    long long m = d.cls_pib[3 * c + i];
                    for (int j = 0; j < 3; ++j) m += (long long)d.cls_piA[9 * c + 3 * i + j] * d.sites[3 * sidx + j];
                    if (m % d.diag[i] != 0) {
                        delete p;
                        return fail(SP_ERR_INVALID, "mapped site not on the zero coset (class %d)", c);
                    }
                    const int z = (int)(m / d.diag[i]);
                    site_off[((size_t)c * n_sites + sidx) * 3 + i] = z;
                    if (kern == d.cls_kernel[c]) {
                        if (first) { p->reach_lo[i] = p->reach_hi[i] = z; }
                        else {
                            p->reach_lo[i] = std::min(p->reach_lo[i], z);
                            p->reach_hi[i] = std::max(p->reach_hi[i], z);
                        }
                    }
                }
                if (kern == d.cls_kernel[c]) first = false;
            }
        }
    }

    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);

    if (d.tp_degree >= 0) {
        int rc = verify_tensor(d, d.tp_degree);
        if (rc != SP_OK) { delete p; return rc; }
        p->kind = SP_KIND_TENSOR_BSPLINE;
        p->tp_degree = d.tp_degree;
        p->name = "tensor_bspline_" + std::to_string(d.tp_degree);
        *out = p;
        return SP_OK;
    }

    const std::vector<uint64_t> words = canonical_words(d, n_sites, n_terms);
    for (const sp::GenEntry* ep : kGenerated) {
        if (d.tp_degree == -2) break;  // caller forces the generic kernel
        if (!ep) continue;
        const sp::GenEntry& e = *ep;
        if (e.blob_len == (int)words.size() && std::memcmp(e.blob, words.data(), words.size() * 8) == 0) {
            p->gen = &e;
            break;
        }
    }
    // the reference's bcc_linear_rd plan (matched word for word above) has a closed form
    // (sp_bcc_linear.cuh); it reads coset cells -2..+2 around floor((x - l)/2)
    if (p->gen && std::strcmp(p->gen->name, "bcc_linear_rd") == 0 && env_int("SP_BCC_TET", 1) != 0) {
        p->bcc_tet = true;
        for (int i = 0; i < 3; ++i) {
            p->reach_lo[i] = std::min(p->reach_lo[i], -2);
            p->reach_hi[i] = std::max(p->reach_hi[i], 2);
        }
    }

    if (p->gen) {
        // plan tables (generated layout, codegen kClsOff / kCubeOff / kSigOff): uint4 class
        // records [N] | unit-cube class-word table (codegen.cube_table, 16 B aligned) | int32
        // sigma[r]; the leading gen->smem_table_bytes are staged into shared memory
        const int sig_bytes = ((d.r * 4) + 15) & ~15;
        const int cube_words = p->gen->cube_tab ? ((p->gen->cube_len + 3) & ~3) : 0;
        const int sig_off = 4 * d.N + cube_words;  // in 32-bit words
        std::vector<uint32_t> blob(sig_off + sig_bytes / 4, 0);
        if (p->gen->cube_tab) std::memcpy(blob.data() + 4 * d.N, p->gen->cube_tab, (size_t)p->gen->cube_len * 4);
        for (int j = 0; j < d.r; ++j) blob[sig_off + j] = (uint32_t)d.sigma[j];
        for (int c = 0; c < d.N; ++c) {
            int perm[3], sign[3], rho[3], tau[3];
            if (!signed_perm(d.cls_T + 9 * c, perm, sign)) { delete p; return fail(SP_ERR_INVALID, "generated plan needs signed-permutation T"); }
            double A[9];
            for (int j = 0; j < 9; ++j) A[j] = d.cls_piA[9 * c + j];
            if (!signed_perm(A, rho, tau)) { delete p; return fail(SP_ERR_INVALID, "generated plan needs signed-permutation piA"); }
            // x: kernel | perm_i << (4+2i) | (sign_i<0) << (10+i) | rho_i << (13+2i) | (tau_i<0) << (19+i)
            //    | (pib_i/d + 4) << (22+3i);   y, z, w: t_0, t_1, t_2 as float bits
            uint32_t x = (uint32_t)d.cls_kernel[c];
            float tf[3];
            for (int i = 0; i < 3; ++i) {
                x |= (uint32_t)perm[i] << (4 + 2 * i);
                x |= (uint32_t)(sign[i] < 0) << (10 + i);
                x |= (uint32_t)rho[i] << (13 + 2 * i);
                x |= (uint32_t)(tau[i] < 0) << (19 + i);
                const double ti = d.cls_t[3 * c + i];
                if (ti != std::floor(ti) || std::fabs(ti) > 1024) { delete p; return fail(SP_ERR_INVALID, "non-integral class shift t"); }
                tf[i] = (float)ti;
                const int pbd = d.cls_pib[3 * c + i] / d.diag[i];
                if (pbd < -4 || pbd > 3) { delete p; return fail(SP_ERR_UNSUPPORTED, "class offset out of range"); }
                x |= (uint32_t)(pbd + 4) << (22 + 3 * i);
            }
            uint32_t* rec = blob.data() + 4 * c;
            rec[0] = x;
            std::memcpy(rec + 1, tf, sizeof tf);
        }
        const uint32_t* dptr = nullptr;
        if (upload(p, blob, &dptr) != SP_OK) { delete p; return SP_ERR_CUDA; }
        p->d_tables = (void*)dptr;
        p->table_bytes = p->gen->smem_table_bytes;  // staged into shared memory
        if (p->table_bytes > (int)(blob.size() * 4)) { delete p; return fail(SP_ERR_INVALID, "plan table layout"); }
        p->kind = SP_KIND_GENERATED;
        p->name = std::string("gen:") + p->gen->name;
        *out = p;
        return SP_OK;
    }

    // generic tables
    sp::GenericTables gt{};
    gt.Q = d.Q; gt.r = d.r; gt.N = d.N; gt.K = d.K; gt.n_sites = n_sites;
    std::vector<int> normals(d.normals, d.normals + d.Q * 3);
    std::vector<double> offsets(d.offsets, d.offsets + d.Q);
    std::vector<int> sigma(d.sigma, d.sigma + d.r);
    std::vector<int> ck(d.cls_kernel, d.cls_kernel + d.N);
    std::vector<double> cT(d.cls_T, d.cls_T + d.N * 9), ct(d.cls_t, d.cls_t + d.N * 3);
    std::vector<int> kgs(d.kernel_group_start, d.kernel_group_start + d.K + 1);
    std::vector<int> gns(d.group_nspan, d.group_nspan + d.n_groups);
    std::vector<int> gss(d.group_site_start, d.group_site_start + d.n_groups + 1);
    std::vector<int> gps(d.group_poly_start, d.group_poly_start + d.n_groups + 1);
    std::vector<int> pts(d.poly_term_start, d.poly_term_start + d.n_polys + 1);
    std::vector<int> tex(d.term_exps, d.term_exps + n_terms * 3);
    std::vector<double> tco(d.term_coeffs, d.term_coeffs + n_terms);
    int rc = SP_OK;
    rc |= upload(p, normals, &gt.normals);
    rc |= upload(p, offsets, &gt.offsets);
    rc |= upload(p, sigma, &gt.sigma);
    rc |= upload(p, ck, &gt.cls_kernel);
    rc |= upload(p, cT, &gt.cls_T);
    rc |= upload(p, ct, &gt.cls_t);
    rc |= upload(p, kgs, &gt.kernel_group_start);
    rc |= upload(p, gns, &gt.group_nspan);
    rc |= upload(p, gss, &gt.group_site_start);
    rc |= upload(p, gps, &gt.group_poly_start);
    rc |= upload(p, site_off, &gt.site_off);
    rc |= upload(p, pts, &gt.poly_term_start);
    rc |= upload(p, tex, &gt.term_exps);
    rc |= upload(p, tco, &gt.term_coeffs);
    if (rc != SP_OK) { delete p; return SP_ERR_CUDA; }
    void* dgt = nullptr;
    if (cudaMalloc(&dgt, sizeof gt) != cudaSuccess || cudaMemcpy(dgt, &gt, sizeof gt, cudaMemcpyHostToDevice) != cudaSuccess) {
        delete p;
        return fail(SP_ERR_CUDA, "generic table upload failed");
    }
    p->allocs.push_back(dgt);
    p->d_tables = dgt;
    p->table_bytes = 0;
    p->kind = SP_KIND_GENERIC;
    p->name = "generic";
    *out = p;
    return SP_OK;
}

void sp_plan_destroy(sp_plan* plan) {
    if (!plan) return;
    for (void* ptr : plan->allocs) cudaFree(ptr);
    delete plan;
}

int sp_plan_kernel_kind(const sp_plan* plan) { return plan ? (int)plan->kind : -1; }
const char* sp_plan_kernel_name(const sp_plan* plan) { return plan ? plan->name.c_str() : ""; }

int sp_eval_launch_count(const sp_plan* plan, int64_t n) { return (plan && n > 0) ? 1 : 0; }

}  // extern "C"

namespace {

// Tuning knobs (environment, read per call): SP_TILE_KB (shared-memory tile budget),
// SP_PPT (points per thread per chunk, 0 = density-based).
// shared-memory tile budget: SP_TILE_KB, else the generated plan's (codegen.tile_budget_kb), else 40 KB
int tile_bytes(const sp_plan* p = nullptr) {
    return env_int("SP_TILE_KB", (p && p->gen && p->gen->tile_kb > 0) ? p->gen->tile_kb : 40) * 1024;
}

unsigned long long* g_stats = nullptr;  // device [4] when sp_debug_stats(1) is on

// Points per thread per chunk from the point density: aim for ~256 unit cells per chunk so
// the staged box (+ halo) stays small; 1..kMaxPPT.
int choose_ppt(const sp_plan* p, const sp_grid_desc* g, int64_t n) {
    double cells = 1.0;
    for (int i = 0; i < 3; ++i) cells *= (double)g->extent[0][i] * p->diag[i];
    const double density = (double)n / std::max(cells, 1.0);
    const double want = 256.0 * density / sp::kThreads;
    int ppt = 1;
    while (ppt < sp::kMaxPPT && ppt * 2 <= want) ppt *= 2;
    const int forced = env_int("SP_PPT", 0);
    if (forced > 0) ppt = std::min(forced, sp::kMaxPPT);
    return ppt;
}

template <typename T>
int build_args(const sp_plan* p, const sp_grid_desc* g, const void* pts, int64_t n, void* out, int32_t* dbg,
               int32_t* err, sp::EvalArgs<T>& a, int& vec) {
    a = sp::EvalArgs<T>{};
    a.grid.M = g->M;
    a.grid.boundary = g->boundary;
    for (int k = 0; k < g->M; ++k) {
        a.grid.data[k] = reinterpret_cast<const T*>(g->data[k]);
        for (int i = 0; i < 3; ++i) {
            if (g->extent[k][i] < 1 || g->extent[k][i] > (1ll << 30)) return fail(SP_ERR_INVALID, "coset extent out of range");
            if (g->origin[k][i] < -(1ll << 30) || g->origin[k][i] > (1ll << 30)) return fail(SP_ERR_INVALID, "coset origin out of range");
            a.grid.ext[k][i] = (int)g->extent[k][i];
            a.grid.org[k][i] = (int)g->origin[k][i];
        }
        if (!g->data[k]) return fail(SP_ERR_INVALID, "null coset array %d", k);
    }
    a.fr.M = p->M;
    for (int i = 0; i < 3; ++i) {
        a.fr.diag[i] = p->diag[i];
        a.fr.dlog2[i] = -1;
        for (int b = 0; b < 30; ++b)
            if ((1 << b) == p->diag[i]) a.fr.dlog2[i] = b;
        a.fr.reach_lo[i] = p->reach_lo[i];
        a.fr.reach_hi[i] = p->reach_hi[i];
    }
    for (int k = 0; k < p->M; ++k)
        for (int i = 0; i < 3; ++i) a.fr.shift[k][i] = p->shifts[k][i];
    a.pts = reinterpret_cast<const T*>(pts);
    a.out = reinterpret_cast<T*>(out);
    a.n = n;
    a.dbg = dbg;
    a.err = err;
    a.tables = p->d_tables;
    a.table_bytes = p->table_bytes;
    a.trec_bytes = p->kind == SP_KIND_GENERATED ? p->gen->trec_bytes : 0;
    // row-vector tile (fp32 tensor-product kernels): +vec*sizeof(T) bytes per tile element
    vec = (p->kind == SP_KIND_TENSOR_BSPLINE && sizeof(T) == 4) ? (p->tp_degree == 1 ? 2 : 4) : 0;
    if (vec) {
        // scalar staging tile + padded row-vector tile (~1.5x the scalar capacity)
        // SP_VPAD=1: bank-conflict-padded row-vector tile (tuning knob; dense measured faster)
        const bool pad = env_int("SP_VPAD", 0) != 0;
        a.tile_cap = tile_bytes(p) / (int)(sizeof(T) * (1 + (pad ? vec * 3 / 2 : vec)));
        a.vec_cap = pad ? a.tile_cap * 3 / 2 : a.tile_cap;
    } else {
        // the closed-form BCC linear plan uses 32^3 fp32 bricks (brick_log2_typed): 80 KB tile
        // for the generic drivers (protocol B) so that those bricks still stage
        a.tile_cap = (p->bcc_tet ? std::max(tile_bytes(p), 80 * 1024) : tile_bytes(p)) / (int)sizeof(T);
        a.vec_cap = 0;
    }
    a.stats = g_stats;
    a.ppt = choose_ppt(p, g, n);
    bool shifted = false;
    for (int k = 0; k < p->M; ++k)
        for (int i = 0; i < 3; ++i) shifted |= p->shifts[k][i] != 0;
    // float32 points: x - l is exact in float64 and floor((x-l)/d) == floordiv(floor(x)-l, d);
    // float64 points may round x - l, so keep one cell of slack around the staged box.
    a.margin = (sizeof(T) == 8 && shifted) ? 1 : 0;
    return SP_OK;
}

template <typename T>
size_t tile_smem(const sp::EvalArgs<T>& a, int vec, size_t esz) {
    return (size_t)((a.table_bytes + 15) & ~15) + (size_t)a.trec_bytes +
           ((((size_t)a.tile_cap + 4) * esz + 15) & ~(size_t)15) +
           (size_t)a.vec_cap * vec * esz;
}

template <typename T>
struct Kernels {
    sp::LaunchFn<T> chunk = nullptr;
    sp::BrickLaunchFn<T> brick = nullptr;
    int (*occ)(size_t) = nullptr;
    int (*bocc)(size_t) = nullptr;
};

template <typename T, class Ev>
Kernels<T> kernels_of() {
    Kernels<T> k;
    k.chunk = &sp::launch_eval<T, Ev>;
    k.brick = &sp::launch_bricks<T, Ev>;
    k.occ = &sp::occupancy_blocks<T, Ev>;
    k.bocc = &sp::occupancy_bricks<T, Ev>;
    return k;
}

template <typename T>
int select_kernels(const sp_plan* p, Kernels<T>& k, bool dbg = false) {
    if (p->bcc_tet && !dbg) {  // class ids (dbg) come from the plan-generated classification
        k = kernels_of<T, sp::BccTetEval<T>>();
        return SP_OK;
    }
    if (p->kind == SP_KIND_TENSOR_BSPLINE) {
        switch (p->tp_degree) {
            case 1: k = kernels_of<T, sp::TensorBSplineEval<T, 1>>(); return SP_OK;
            case 2: k = kernels_of<T, sp::TensorBSplineEval<T, 2>>(); return SP_OK;
            case 3: k = kernels_of<T, sp::TensorBSplineEval<T, 3>>(); return SP_OK;
            default: return fail(SP_ERR_UNSUPPORTED, "tensor degree");
        }
    }
    if (p->kind == SP_KIND_GENERATED) {
        if constexpr (sizeof(T) == 4) {
            k.chunk = p->gen->launch_f32; k.occ = p->gen->occ_f32; k.brick = p->gen->brick_f32; k.bocc = p->gen->bocc_f32;
        } else {
            k.chunk = p->gen->launch_f64; k.occ = p->gen->occ_f64; k.brick = p->gen->brick_f64; k.bocc = p->gen->bocc_f64;
        }
        return SP_OK;
    }
    k = kernels_of<T, sp::GenericEval<T>>();
    return SP_OK;
}

template <typename T>
int eval_typed(const sp_plan* p, const sp_grid_desc* g, const void* pts, int64_t n, void* out, int32_t* dbg,
               int32_t* err, cudaStream_t st) {
    sp::EvalArgs<T> a;
    int vec = 0;
    int rc = build_args<T>(p, g, pts, n, out, dbg, err, a, vec);
    if (rc != SP_OK) return rc;
    Kernels<T> k;
    if ((rc = select_kernels<T>(p, k, dbg != nullptr)) != SP_OK) return rc;
    const int chunk_pts = sp::kThreads * a.ppt;
    const size_t smem = tile_smem(a, vec, sizeof(T)) +
                        (size_t)((chunk_pts * 3 * sizeof(T) + 15) & ~15);
    const long long nchunks = (n + chunk_pts - 1) / chunk_pts;
    const long long cap = (long long)p->num_sms * k.occ(smem);
    const int blocks = (int)std::max<long long>(1, std::min<long long>(nchunks, cap));
    cudaError_t e = k.chunk(a, blocks, smem, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SP_OK;
}

// Largest brick edge 2^b (unit cells) whose staged box (all cosets, + reach, + margin) fits
// the tile; -1 when even 4^3 bricks do not fit.
template <typename T>
int brick_log2_typed(const sp_plan* p) {
    // closed-form BCC linear kernel (sp_bcc_linear.cuh): 32^3 bricks for fp32 (64 KB tile,
    // barriers and staging amortised over ~8x more points than 16^3); SP_BCC_TET_L2B overrides
    if (p->bcc_tet && env_int("SP_BCC_TET_BRICK", 1) != 0) return env_int("SP_BCC_TET_L2B", sizeof(T) == 4 ? 5 : 4);
    const int vec = (p->kind == SP_KIND_TENSOR_BSPLINE && sizeof(T) == 4) ? (p->tp_degree == 1 ? 2 : 4) : 0;
    const long long cap = tile_bytes(p) / (long long)(sizeof(T) * (1 + vec * 3 / 2));
    bool shifted = false;
    for (int k = 0; k < p->M; ++k)
        for (int i = 0; i < 3; ++i) shifted |= p->shifts[k][i] != 0;
    const int margin = (sizeof(T) == 8 && shifted) ? 1 : 0;
    for (int b = 6; b >= 2; --b) {
        const int B = 1 << b;
        long long total = 0;
        for (int k = 0; k < p->M; ++k) {
            long long vol = 1;
            for (int i = 0; i < 3; ++i) {
                const int d = p->diag[i], l = p->shifts[k][i];
                auto fdiv = [](long long a, long long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
                // coset cells covered by the unit cells [0, B-1] of an aligned brick
                const long long cells = fdiv(B - 1 - l, d) - fdiv(-l, d) + 1;
                const long long ext = cells + (p->reach_hi[i] - p->reach_lo[i]) + 2 * margin;
                vol *= ext;
            }
            total += vol;
        }
        if (total <= cap) return b;
    }
    return -1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    // initialised once, thread-safely (function-local static)
    static const EncodeTiledFn fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(f);
        return (EncodeTiledFn) nullptr;
    }();
    return fn;
}

template <int DEG, int S0 = 0, int S1 = 0, class G = sp::TmaGeom<>>
cudaError_t launch_tma(const sp::EvalArgs<float>& a, const CUtensorMap& map, const long long* bstart, int nbricks,
                       int log2b, int bx, int by, int bz, int vx, int vy, size_t smem, int num_sms, cudaStream_t st) {
    using Ev = sp::TensorBSplineEval<float, DEG, S0, S1>;
    auto kern = sp::brick_kernel_tma<float, Ev, G>;
    const int per_sm = sp::cached_occupancy(kern, smem);  // also sets the dynamic smem limit
    const int blocks = std::max(1, std::min(nbricks, num_sms * per_sm));
    kern<<<blocks, sp::kThreads, smem, st>>>(a, map, bstart, nbricks, log2b, bx, by, bz, vx, vy);
    return cudaGetLastError();
}

// Pitches of the TMA box (= the row-vector tile) that keep the row loads of Morton-adjacent
// cells in different shared-memory bank groups: two lanes of one load phase (8 lanes for
// LDS.128, 16 for LDS.64) reading different rows whose float offsets differ by a multiple of
// 32 banks serialise.  Lanes hold consecutive Morton-ordered points, so the rows they read
// belong to Morton-consecutive cells; score each candidate (bx, by) by the cell pairs at
// Morton distance 1 and 2 inside a brick whose row offset is a multiple of the phase's slot
// count, and take the cheapest (then smallest) box.
void choose_box_pitch_uncached(int need_x, int need_y, int B, int slots, int xstep, int& bx, int& by);

// memoised: the search is O(B^3 * candidates) host work, far too slow to repeat per launch
void choose_box_pitch(int need_x, int need_y, int B, int slots, int xstep, int& bx, int& by) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int>, std::pair<int, int>> memo;
    const auto key = std::make_tuple(need_x, need_y, B, slots, xstep);
    std::lock_guard<std::mutex> lock(mu);
    auto it = memo.find(key);
    if (it == memo.end()) {
        std::pair<int, int> v;
        choose_box_pitch_uncached(need_x, need_y, B, slots, xstep, v.first, v.second);
        it = memo.emplace(key, v).first;
    }
    bx = it->second.first;
    by = it->second.second;
}

void choose_box_pitch_uncached(int need_x, int need_y, int B, int slots, int xstep, int& bx, int& by) {
    auto spread = [](int v) {
        int o = 0;
        for (int i = 0; i < 5; ++i) o |= ((v >> i) & 1) << (3 * i);
        return o;
    };
    std::vector<std::pair<int, int>> cells;  // (morton, packed zyx)
    for (int z = 0; z < B; ++z)
        for (int y = 0; y < B; ++y)
            for (int x = 0; x < B; ++x) cells.push_back({spread(x) | spread(y) << 1 | spread(z) << 2, (z << 10) | (y << 5) | x});
    std::sort(cells.begin(), cells.end());
    long best = -1;
    const int bx0 = (need_x + xstep - 1) / xstep * xstep;
    for (int cx = bx0; cx <= bx0 + 12 && cx <= 256; cx += xstep)
        for (int cy = need_y; cy <= need_y + 4 && cy <= 256; ++cy) {
            long cost = 0;
            for (size_t i = 0; i < cells.size(); ++i)
                for (size_t d = 1; d <= 2 && i + d < cells.size(); ++d) {
                    const int a = cells[i].second, b = cells[i + d].second;
                    const long D = (long)((b >> 10) - (a >> 10)) * cx * cy + (long)(((b >> 5) & 31) - ((a >> 5) & 31)) * cx +
                                   ((b & 31) - (a & 31));
                    cost += (D != 0 && D % slots == 0);
                }
            const long score = cost * (1l << 24) + (long)cx * cy;
            if (best < 0 || score < best) {
                best = score;
                bx = cx;
                by = cy;
            }
        }
}

// TMA-staged brick path: fp32 single-coset tensor-product plans, 'zero' boundary, 16-byte
// aligned rows.  Returns 1 when launched, 0 when not applicable, < 0 on error.
int try_bricks_tma(const sp_plan* p, const sp_grid_desc* g, const sp::EvalArgs<float>& a, const int64_t* bstart,
                   int nbricks, int log2b, cudaStream_t st) {
    if (env_int("SP_TMA", 1) == 0) return 0;
    if (p->kind != SP_KIND_TENSOR_BSPLINE || g->M != 1 || g->boundary != SP_ZERO || a.margin != 0) return 0;
    if (p->tp_degree != 1 && p->tp_degree != 3) return 0;
    const long long e0 = g->extent[0][0], e1 = g->extent[0][1], e2 = g->extent[0][2];
    if ((e2 * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(g->data[0]) & 15) != 0) return 0;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return 0;
    const int B = 1 << log2b;
    const int span[3] = {B + p->reach_hi[0] - p->reach_lo[0], B + p->reach_hi[1] - p->reach_lo[1],
                         B + p->reach_hi[2] - p->reach_lo[2]};
    // innermost TMA start coordinate must be 16-byte aligned: start rounded down, box widened
    const int vec = p->tp_degree == 1 ? 2 : 4;
    // SP_BOXPAD: 0 = dense box and row-vector tile, 1 = conflict-free TMA box pitches (the
    // tile copy stays 1:1), 2 = dense TMA box, conflict-free row-vector tile pitches
    const int boxpad = env_int("SP_BOXPAD", 2);
    int bx = (span[2] + 3 + 3) & ~3, by = span[1];
    if (boxpad == 1) choose_box_pitch(span[2] + 3, span[1], B, 128 / (vec * 4), 4, bx, by);
    int vx = bx, vy = by;
    if (boxpad == 2) choose_box_pitch(bx, by, B, 128 / (vec * 4), 1, vx, vy);
    const int bz = span[0];
    if (bx > 256 || by > 256 || bz > 256) return 0;
    const int boxv = bx * by * bz;
    const size_t smem = 2 * (size_t)((boxv * 4 + 127) & ~127) + (size_t)vx * vy * bz * vec * 4;
    if (smem > 100 * 1024) return 0;
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)e2, (cuuint64_t)e1, (cuuint64_t)e0};
    const cuuint64_t strides[2] = {(cuuint64_t)(e2 * 4), (cuuint64_t)(e2 * e1 * 4)};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(g->data[0]), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 0;
    const long long* bs = reinterpret_cast<const long long*>(bstart);
    // the headline configuration (tricubic, 8^3 bricks -> 18 x 11 conflict-free pitches) has a
    // specialisation with compile-time tile pitches; SP_TMA_FIXED=0 disables it
    const bool fixed = p->tp_degree == 3 && log2b == 3 && bx == 16 && by == 11 && bz == 11 && vx == 18 && vy == 11 &&
                       env_int("SP_TMA_FIXED", 1) != 0;
    cudaError_t e = p->tp_degree == 1
                        ? launch_tma<1>(a, map, bs, nbricks, log2b, bx, by, bz, vx, vy, smem, p->num_sms, st)
                    : fixed ? launch_tma<3, 18 * 11, 18, sp::TmaGeom<3, 16, 11, 11, 18, 11>>(a, map, bs, nbricks, log2b, bx, by,
                                                                                          bz, vx, vy, smem, p->num_sms, st)
                            : launch_tma<3>(a, map, bs, nbricks, log2b, bx, by, bz, vx, vy, smem, p->num_sms, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "TMA brick kernel launch: %s", cudaGetErrorString(e));
    return 1;
}

// Closed-form brick kernel of the BCC linear box spline (sp_bcc_linear.cuh): the plan is the
// reference's bcc_linear_rd (matched word for word against the generated registry entry),
// brick-order points read directly (no permutation), 16-byte aligned points and results.
// Returns 1 when launched, 0 when not applicable, < 0 on error.  SP_BCC_TET=0 disables.
template <typename T>
int try_bricks_bcc_tet(const sp_plan* p, const sp::EvalArgs<T>& a, const int64_t* bstart, int nbricks, int log2b,
                       cudaStream_t st) {
    if (!p->bcc_tet || env_int("SP_BCC_TET_BRICK", 1) == 0) return 0;
    if (a.in_index32 || a.out_index || a.out_index32 || a.dbg) return 0;
    if ((reinterpret_cast<uintptr_t>(a.pts) & 15) || (reinterpret_cast<uintptr_t>(a.out) & 15)) return 0;
    if (log2b < 3 || log2b > 5) return 0;
    const long long* bs = reinterpret_cast<const long long*>(bstart);
    const int E = (1 << log2b) / 2 + 2;
    // SP_BCC_TET_VARIANT (tuning): 0 = lean tile path, two point groups in flight per thread
    // (bcc_tet_brick_kernel_v2, default); 3 = the round-2 kernel (register prefetch of the
    // next quad, per-point brick test); 1 = no prefetch, 4 CTAs/SM; 2 = prefetch +
    // double-buffered tile; 4 = the lean kernel at 4 CTAs/SM (fp32).  All give identical values.
    static const int variant = env_int("SP_BCC_TET_VARIANT", 0);
    const bool db = variant == 2;
    const size_t smem = (db ? 4 : 2) * (size_t)E * E * E * sizeof(T);  // two cosets (x2 double-buffered)
    // the round-2 kernel: variant 3, or float64 with SP_BCC_TET_LEAN64=0 (the lean kernel's
    // 2-point float64 groups: 106.7 -> 114.9 Gpts/s at C3)
    static const bool lean64 = env_int("SP_BCC_TET_LEAN64", 1) != 0;
    const bool old = variant == 3 || (sizeof(T) == 8 && !lean64);
    auto kern = log2b == 3   ? (old ? sp::bcc_tet_brick_kernel<T, 3> : sp::bcc_tet_brick_kernel_v2<T, 3>)
                : log2b == 4 ? (old ? sp::bcc_tet_brick_kernel<T, 4> : sp::bcc_tet_brick_kernel_v2<T, 4>)
                : variant == 1 ? sp::bcc_tet_brick_kernel<T, 5, false, sizeof(T) == 4 ? 4 : 2>
                : variant == 2 ? sp::bcc_tet_brick_kernel<T, 5, true, sizeof(T) == 4 ? 3 : 2, true>
                : variant == 4 ? sp::bcc_tet_brick_kernel_v2<T, 5, sizeof(T) == 4 ? 4 : 3>
                : old        ? sp::bcc_tet_brick_kernel<T, 5>
                               : sp::bcc_tet_brick_kernel_v2<T, 5>;
    const int per_sm = sp::cached_occupancy(kern, smem);
    const int blocks = std::max(1, std::min(nbricks, p->num_sms * per_sm));
    kern<<<blocks, sp::kThreads, smem, st>>>(a, bs, nbricks);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "BCC linear brick kernel launch: %s", cudaGetErrorString(e));
    return 1;
}

template <typename T>
int eval_bricks_typed(const sp_plan* p, const sp_grid_desc* g, const void* pts, int64_t n, const int64_t* bstart,
                      int32_t nbricks, int32_t log2b, const int64_t* out_index, void* out, int32_t* err,
                      cudaStream_t st, const int32_t* nbricks_dev = nullptr, const int32_t* out_index32 = nullptr,
                      const int32_t* in_index32 = nullptr) {
    sp::EvalArgs<T> a;
    int vec = 0;
    int rc = build_args<T>(p, g, pts, n, out, nullptr, err, a, vec);
    if (rc != SP_OK) return rc;
    a.out_index = reinterpret_cast<const long long*>(out_index);
    a.out_index32 = out_index32;
    a.in_index32 = in_index32;
    a.nbricks_dev = nbricks_dev;
    a.prefetch_pts = env_int("SP_PREFETCH_PTS", 1);
    a.plain_pts = env_int("SP_PLAIN_PTS", 1);
    // float64 tensor-product tiles are read as scalar rows (LDS.64, 16 bank slots): widen the
    // staged box so that Morton-adjacent cells fall in different bank slots (SP_F64_PAD=0: off)
    if (sizeof(T) == 8 && p->kind == SP_KIND_TENSOR_BSPLINE && g->M == 1 && log2b >= 2 && log2b <= 4 &&
        env_int("SP_F64_PAD", 1) != 0) {
        const int B = 1 << log2b;
        const int need_x = B + p->reach_hi[2] - p->reach_lo[2], need_y = B + p->reach_hi[1] - p->reach_lo[1];
        int bx = need_x, by = need_y;
        choose_box_pitch(need_x, need_y, B, 16, 1, bx, by);
        a.box_pad[2] = bx - need_x;
        a.box_pad[1] = by - need_y;
    }
    if constexpr (sizeof(T) == 4) {
        const int t = try_bricks_tma(p, g, a, bstart, nbricks, log2b, st);
        if (t != 0) return t > 0 ? SP_OK : t;
    }
    {
        const int t = try_bricks_bcc_tet<T>(p, a, bstart, nbricks, log2b, st);
        if (t != 0) return t > 0 ? SP_OK : t;
    }
    Kernels<T> k;
    if ((rc = select_kernels<T>(p, k)) != SP_OK) return rc;
    const size_t smem = tile_smem(a, vec, sizeof(T));
    const long long cap = (long long)p->num_sms * k.bocc(smem);
    const int blocks = (int)std::max<long long>(1, std::min<long long>(nbricks, cap));
    cudaError_t e = k.brick(a, reinterpret_cast<const long long*>(bstart), nbricks, log2b, blocks, smem, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SP_OK;
}

int check_grid(const sp_plan* p, const sp_grid_desc* g, int32_t dtype) {
    if (!g) return fail(SP_ERR_INVALID, "null grid");
    if (g->s != p->s || g->M != p->M) return fail(SP_ERR_MISMATCH, "grid decomposition does not match the plan header");
    for (int i = 0; i < 3; ++i)
        if (g->diag[i] != p->diag[i]) return fail(SP_ERR_MISMATCH, "grid decomposition does not match the plan header");
    for (int k = 0; k < p->M; ++k)
        for (int i = 0; i < 3; ++i)
            if (g->shifts[k][i] != p->shifts[k][i]) return fail(SP_ERR_MISMATCH, "grid decomposition does not match the plan header");
    if (g->dtype != dtype) return fail(SP_ERR_INVALID, "grid dtype must equal the point dtype");
    if (g->boundary < SP_ZERO || g->boundary > SP_MIRROR) return fail(SP_ERR_INVALID, "unknown boundary policy %d", g->boundary);
    return SP_OK;
}

}  // namespace

extern "C" int sp_eval(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                       void* out, int32_t* dbg, int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0) return fail(SP_ERR_INVALID, "negative n");
    if (n == 0) return SP_OK;
    if (!pts || !out) return fail(SP_ERR_INVALID, "null points or output");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32) return eval_typed<float>(plan, grid, pts, n, out, dbg, err_flag, st);
    if (dtype == SP_F64) return eval_typed<double>(plan, grid, pts, n, out, dbg, err_flag, st);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

// Texture-filtered evaluation of a generated plan (called by sp_eval_texture, sp_texture.cu):
// `g` describes the cosets' extents / origins / policy (data pointers unused), `targs` the
// texture objects.
namespace sp {
int eval_texture_generated(const sp_plan* p, const sp_grid_desc* g, const TexArgs& targs, const void* pts, int64_t n,
                           void* out, int32_t* err, cudaStream_t st) {
    if (p->kind != SP_KIND_GENERATED || !p->gen || !p->gen->tex_f32)
        return fail(SP_ERR_UNSUPPORTED, "texture variant: no compiled texture kernel for this plan");
    EvalArgs<float> a;
    int vec = 0;
    int rc = build_args<float>(p, g, pts, n, out, nullptr, err, a, vec);
    if (rc != SP_OK) return rc;
    cudaError_t e = p->gen->tex_f32(a, targs, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "texture kernel launch: %s", cudaGetErrorString(e));
    return SP_OK;
}
}  // namespace sp

extern "C" int sp_debug_stats(int enable, uint64_t* out) {
    if (out) {
        if (g_stats) {
            SP_CUDA(cudaMemcpy(out, g_stats, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        } else {
            for (int i = 0; i < 4; ++i) out[i] = 0;
        }
    }
    if (enable && !g_stats) {
        SP_CUDA(cudaMalloc(&g_stats, 4 * sizeof(unsigned long long)));
    }
    if (enable) SP_CUDA(cudaMemset(g_stats, 0, 4 * sizeof(unsigned long long)));
    if (!enable && g_stats) {
        cudaFree(g_stats);
        g_stats = nullptr;
    }
    return SP_OK;
}

extern "C" int sp_brick_log2(const sp_plan* plan, int32_t dtype) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    if (dtype == SP_F32) return brick_log2_typed<float>(plan);
    if (dtype == SP_F64) return brick_log2_typed<double>(plan);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

extern "C" int sp_eval_bricks(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                              const int64_t* brick_start, int32_t n_bricks, int32_t log2_brick,
                              const int64_t* out_index, void* out, int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0 || n_bricks < 0) return fail(SP_ERR_INVALID, "negative size");
    if (n == 0 || n_bricks == 0) return SP_OK;
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (!pts || !out || !brick_start) return fail(SP_ERR_INVALID, "null points, output or brick_start");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        return eval_bricks_typed<float>(plan, grid, pts, n, brick_start, n_bricks, log2_brick, out_index, out, err_flag,
                                        st);
    if (dtype == SP_F64)
        return eval_bricks_typed<double>(plan, grid, pts, n, brick_start, n_bricks, log2_brick, out_index, out, err_flag,
                                         st);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

extern "C" int sp_eval_bricks_dev(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n,
                                  int32_t dtype, const int64_t* brick_start, const int32_t* n_bricks_dev,
                                  int32_t n_bricks_cap, int32_t log2_brick, const int64_t* out_index, void* out,
                                  int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0 || n_bricks_cap < 0) return fail(SP_ERR_INVALID, "negative size");
    if (n == 0 || n_bricks_cap == 0) return SP_OK;
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (!pts || !out || !brick_start || !n_bricks_dev) return fail(SP_ERR_INVALID, "null points, output or brick runs");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        return eval_bricks_typed<float>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, out_index, out,
                                        err_flag, st, n_bricks_dev);
    if (dtype == SP_F64)
        return eval_bricks_typed<double>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, out_index, out,
                                         err_flag, st, n_bricks_dev);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

extern "C" int sp_eval_sync(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                            void* out, void* stream) {
    int32_t* d_err = nullptr;
    SP_CUDA(cudaMalloc(&d_err, sizeof(int32_t)));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaMemsetAsync(d_err, 0, sizeof(int32_t), st);
    int rc = sp_eval(plan, grid, pts, n, dtype, out, nullptr, d_err, stream);
    int32_t h_err = 0;
    if (rc == SP_OK) {
        cudaError_t e = cudaMemcpyAsync(&h_err, d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(SP_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
    }
    cudaFree(d_err);
    if (rc == SP_OK && h_err) rc = fail(SP_ERR_SENTINEL, "sigma sentinel hit in batch evaluation");
    return rc;
}

// ---------------------------------------------------------------------------------------
// Point-order utilities

namespace {

__device__ __forceinline__ uint64_t spread3(uint32_t v) {
    // 21 bits -> every third bit
    uint64_t x = v & 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

template <typename T>
__global__ void morton_kernel(const T* __restrict__ pts, long long n, uint64_t* __restrict__ keys) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // bias so that cells in [-2^20, 2^20) map monotonically to [0, 2^21)
            const int f = sp::clamp_cell(pts[3 * i + a]);
            const int b = min(max(f + (1 << 20), 0), (1 << 21) - 1);
            c[a] = (uint32_t)b;
        }
        // axis 2 (fastest array axis) in the lowest bit
        keys[i] = spread3(c[2]) | (spread3(c[1]) << 1) | (spread3(c[0]) << 2);
    }
}

// 30-bit Morton keys of cells relative to lo (each axis clamped to [0, 2^bits)), for fast
// 32-bit radix sorts when the batch's bounding box is small (<= 1024 cells per axis).
template <typename T>
__global__ void morton32_kernel(const T* __restrict__ pts, long long n, int lo0, int lo1, int lo2, int bits,
                                int* __restrict__ keys) {
    const int hi = (1 << bits) - 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int c0 = min(max(sp::clamp_cell(pts[3 * i]) - lo0, 0), hi);
        const int c1 = min(max(sp::clamp_cell(pts[3 * i + 1]) - lo1, 0), hi);
        const int c2 = min(max(sp::clamp_cell(pts[3 * i + 2]) - lo2, 0), hi);
        keys[i] = (int)(spread3((uint32_t)c2) | (spread3((uint32_t)c1) << 1) | (spread3((uint32_t)c0) << 2));
    }
}

template <typename T>
__global__ void scatter_kernel(const T* __restrict__ src, const int64_t* __restrict__ perm, long long n, T* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[perm[i]] = src[i];
}

template <typename T>
__global__ void gather_points_kernel(const T* __restrict__ pts, const int64_t* __restrict__ perm, long long n, T* __restrict__ dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long j = perm[i];
        dst[3 * i] = pts[3 * j];
        dst[3 * i + 1] = pts[3 * j + 1];
        dst[3 * i + 2] = pts[3 * j + 2];
    }
}

__global__ void iota32_kernel(int* __restrict__ v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = (int)i;
}

template <typename T>
__global__ void gather_points32_kernel(const T* __restrict__ pts, const int* __restrict__ perm, long long n,
                                       T* __restrict__ dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long j = perm[i];
        dst[3 * i] = pts[3 * j];
        dst[3 * i + 1] = pts[3 * j + 1];
        dst[3 * i + 2] = pts[3 * j + 2];
    }
}

int grid_for(int64_t n) {
    long long b = (n + 255) / 256;
    return (int)std::max<long long>(1, std::min<long long>(b, 148ll * 16));
}

}  // namespace

// Brick runs of Morton-ordered points without a host round trip: brick_start[0..count) =
// indices whose brick id (key >> 3*log2b) differs from the previous point's, then
// brick_start[count] = n, count written to device memory (CUB stream compaction).
struct BrickHead {
    const uint64_t* keys;
    int shift;
    __host__ __device__ bool operator()(long long i) const {
        return i == 0 || (keys[i] >> shift) != (keys[i - 1] >> shift);
    }
};

__global__ void brick_runs_tail(long long n, const int32_t* count, int64_t* brick_start) { brick_start[*count] = n; }

// Brick heads straight from Morton-ordered points (sp_brick_runs_points): two consecutive
// points share a brick iff their clamped, biased unit cells (morton_kernel's key inputs)
// agree after >> log2b on every axis — the same test as comparing their Morton keys >> 3*log2b,
// without building the keys.
template <typename T>
__device__ __forceinline__ uint32_t brick_coord(T v, int log2b) {
    return (uint32_t)min(max(sp::clamp_cell(v) + (1 << 20), 0), (1 << 21) - 1) >> log2b;
}
template <typename T>
struct BrickHeadPts {
    const T* pts;
    int log2b;
    __host__ __device__ bool operator()(long long i) const {
#ifdef __CUDA_ARCH__
        if (i == 0) return true;
        const T* p = pts + 3 * i;
        return brick_coord(p[0], log2b) != brick_coord(p[-3], log2b) ||
               brick_coord(p[1], log2b) != brick_coord(p[-2], log2b) ||
               brick_coord(p[2], log2b) != brick_coord(p[-1], log2b);
#else
        return i == 0;
#endif
    }
};

extern "C" int64_t sp_brick_runs_temp_bytes(int64_t n) {
    if (n <= 0 || n >= (1ll << 31)) return 0;
    size_t bytes = 0;
    thrust::counting_iterator<long long> idx(0);
    const BrickHead head{nullptr, 0};
    if (cub::DeviceSelect::If(nullptr, bytes, idx, static_cast<int64_t*>(nullptr), static_cast<int32_t*>(nullptr),
                              (int)n, head) != cudaSuccess)
        return -1;
    return (int64_t)bytes;
}

// Brick runs of Morton-ordered points in three light passes: (1) one thread per point
// computes its brick coordinates, gets the previous point's from the neighbouring lane
// (shuffle; lane 0 reads it), flags "first point of its brick", and a warp ballot packs 32
// flags into a word, counted per group of 8,192 points; (2) an exclusive scan of the group
// counts; (3) one thread per word writes the indices of its set bits at the group offset +
// the prefix of the group's earlier words.  The points are read once (coalesced) and 1 bit
// per point after that; CUB's select over a point-reading predicate needed 0.92 ms per 1e8.
constexpr int kRunGroup = 8192;  // points per count group = 256 words
template <typename T>
__global__ void brick_head_bits_kernel(const T* __restrict__ pts, long long n, int log2b, uint32_t* __restrict__ bits,
                                       int* __restrict__ group_count) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    if (i < n) {
        c0 = brick_coord(pts[3 * i], log2b);
        c1 = brick_coord(pts[3 * i + 1], log2b);
        c2 = brick_coord(pts[3 * i + 2], log2b);
    }
    uint32_t p0 = __shfl_up_sync(0xffffffffu, c0, 1), p1 = __shfl_up_sync(0xffffffffu, c1, 1),
             p2 = __shfl_up_sync(0xffffffffu, c2, 1);
    if (lane == 0 && i > 0 && i < n) {
        p0 = brick_coord(pts[3 * i - 3], log2b);
        p1 = brick_coord(pts[3 * i - 2], log2b);
        p2 = brick_coord(pts[3 * i - 1], log2b);
    }
    const bool h = i < n && (i == 0 || c0 != p0 || c1 != p1 || c2 != p2);
    const uint32_t w = __ballot_sync(0xffffffffu, h);
    if (lane == 0) {
        bits[i >> 5] = w;
        if (w) atomicAdd(group_count + (i / kRunGroup), __popc(w));
    }
}

// The same bits, four points per thread: three 16-byte loads (fp32; six for fp64) keep four
// times the bytes in flight (the one-point-per-thread form reached 2.6 TB/s); each lane's four
// flags form a nibble, eight lanes OR their nibbles into one 32-point word.  Requires a
// 16-byte aligned point array (the host falls back otherwise).
template <typename T>
__global__ void brick_head_bits4_kernel(const T* __restrict__ pts, long long n, long long nwords, int log2b,
                                        uint32_t* __restrict__ bits, int* __restrict__ group_count) {
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // quad index
    const long long i0 = q * 4;
    const int lane = threadIdx.x & 31;
    uint32_t c[4][3];
    T v[12];
    if (i0 + 4 <= n) {
        if constexpr (sizeof(T) == 4) {
            const float4* src = reinterpret_cast<const float4*>(pts + 3 * i0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float4 t = __ldg(src + k);
                v[4 * k] = t.x;
                v[4 * k + 1] = t.y;
                v[4 * k + 2] = t.z;
                v[4 * k + 3] = t.w;
            }
        } else {
            const double2* src = reinterpret_cast<const double2*>(pts + 3 * i0);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const double2 t = __ldg(src + k);
                v[2 * k] = t.x;
                v[2 * k + 1] = t.y;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 12; ++k) v[k] = i0 + k / 3 < n ? pts[3 * i0 + k] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int a = 0; a < 3; ++a) c[u][a] = brick_coord(v[3 * u + a], log2b);
    // previous point of this lane's first one: the last point of the previous lane
    uint32_t p0 = __shfl_up_sync(0xffffffffu, c[3][0], 1), p1 = __shfl_up_sync(0xffffffffu, c[3][1], 1),
             p2 = __shfl_up_sync(0xffffffffu, c[3][2], 1);
    if (lane == 0 && i0 > 0 && i0 < n) {
        p0 = brick_coord(pts[3 * i0 - 3], log2b);
        p1 = brick_coord(pts[3 * i0 - 2], log2b);
        p2 = brick_coord(pts[3 * i0 - 1], log2b);
    }
    uint32_t nib = 0;
    if (i0 < n) {
        nib |= (i0 == 0 || c[0][0] != p0 || c[0][1] != p1 || c[0][2] != p2) ? 1u : 0u;
#pragma unroll
        for (int u = 1; u < 4; ++u)
            nib |= (i0 + u < n && (c[u][0] != c[u - 1][0] || c[u][1] != c[u - 1][1] || c[u][2] != c[u - 1][2]))
                       ? (1u << u)
                       : 0u;
    }
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    const long long wd = i0 >> 5;  // 8 lanes x 4 points = one 32-point word
    if ((lane & 7) == 0 && wd < nwords) {
        bits[wd] = w;
        if (w) atomicAdd(group_count + (i0 / kRunGroup), __popc(w));
    }
}

__global__ void brick_head_write_kernel(const uint32_t* __restrict__ bits, long long nwords,
                                        const int* __restrict__ group_off, const int* __restrict__ group_count,
                                        int ngroups, int64_t* __restrict__ brick_start, int32_t* __restrict__ n_bricks) {
    // one block (256 threads) per group of 256 words; thread = word
    __shared__ int warp_sum[8];
    const long long wd = blockIdx.x * 256ll + threadIdx.x;
    const uint32_t w = wd < nwords ? bits[wd] : 0u;
    const int c = __popc(w);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) before += k < wid ? warp_sum[k] : 0;
    long long pos = (long long)group_off[blockIdx.x] + before + incl - c;
    uint32_t m = w;
    while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        brick_start[pos++] = wd * 32 + b;
    }
    if ((int)blockIdx.x == ngroups - 1 && threadIdx.x == 0) *n_bricks = group_off[blockIdx.x] + group_count[blockIdx.x];
}

namespace {
size_t align256_(size_t v) { return (v + 255) & ~(size_t)255; }
// scratch: bits [n/32 words] | group counts | group offsets | scan temp
size_t brick_runs_points_bytes(int64_t n) {
    const long long ng = (n + kRunGroup - 1) / kRunGroup;
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, static_cast<int*>(nullptr), static_cast<int*>(nullptr), (int)ng);
    return align256_((size_t)ng * kRunGroup / 8) + 2 * align256_((size_t)ng * 4) + scan;
}
}  // namespace

extern "C" int64_t sp_brick_runs_points_temp_bytes(int64_t n) {
    if (n <= 0 || n >= (1ll << 31)) return 0;
    return (int64_t)brick_runs_points_bytes(n);
}

extern "C" int sp_brick_runs_points(const void* pts, int64_t n, int32_t dtype, int32_t log2_brick,
                                    int64_t* brick_start, int32_t* n_bricks, void* temp, int64_t temp_bytes,
                                    void* stream) {
    if (n < 0 || n >= (1ll << 31)) return fail(SP_ERR_INVALID, "brick runs: n out of range");
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (dtype != SP_F32 && dtype != SP_F64) return fail(SP_ERR_INVALID, "unknown dtype");
    if ((n > 0 && !pts) || !brick_start || !n_bricks) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) {
        SP_CUDA(cudaMemsetAsync(n_bricks, 0, sizeof(int32_t), st));
        SP_CUDA(cudaMemsetAsync(brick_start, 0, sizeof(int64_t), st));
        return SP_OK;
    }
    const long long ng = (n + kRunGroup - 1) / kRunGroup;
    const long long nwords = ng * (kRunGroup / 32);
    const size_t need = brick_runs_points_bytes(n);
    void* tmp = temp;
    if (!tmp || (size_t)temp_bytes < need) {
        tmp = nullptr;
        SP_CUDA(cudaMallocAsync(&tmp, need, st));
    }
    unsigned char* base = static_cast<unsigned char*>(tmp);
    const size_t bits_bytes = align256_((size_t)ng * kRunGroup / 8);
    uint32_t* bits = reinterpret_cast<uint32_t*>(base);
    int* cnt = reinterpret_cast<int*>(base + bits_bytes);
    int* off = reinterpret_cast<int*>(base + bits_bytes + align256_((size_t)ng * 4));
    void* scan_tmp = base + bits_bytes + 2 * align256_((size_t)ng * 4);
    size_t scan_bytes = need - (bits_bytes + 2 * align256_((size_t)ng * 4));
    cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)ng * 4, st);
    const unsigned nblk = (unsigned)(nwords * 32 / sp::kThreads);  // covers the padded groups
    const bool quads = (reinterpret_cast<uintptr_t>(pts) & 15) == 0 && env_int("SP_RUNS_QUADS", 1);
    if (e == cudaSuccess && quads) {
        // one thread per 4 points over every padded word of every group
        const unsigned nq = (unsigned)((nwords * 8 + sp::kThreads - 1) / sp::kThreads);
        if (dtype == SP_F32)
            brick_head_bits4_kernel<float><<<nq, sp::kThreads, 0, st>>>((const float*)pts, n, nwords, log2_brick, bits,
                                                                        cnt);
        else
            brick_head_bits4_kernel<double><<<nq, sp::kThreads, 0, st>>>((const double*)pts, n, nwords, log2_brick, bits,
                                                                         cnt);
        e = cudaGetLastError();
    } else if (e == cudaSuccess) {
        if (dtype == SP_F32)
            brick_head_bits_kernel<float><<<nblk, sp::kThreads, 0, st>>>((const float*)pts, n, log2_brick, bits, cnt);
        else
            brick_head_bits_kernel<double><<<nblk, sp::kThreads, 0, st>>>((const double*)pts, n, log2_brick, bits, cnt);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, off, (int)ng, st);
    if (e == cudaSuccess) {
        brick_head_write_kernel<<<(unsigned)ng, 256, 0, st>>>(bits, nwords, off, cnt, (int)ng, brick_start, n_bricks);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        brick_runs_tail<<<1, 1, 0, st>>>(n, n_bricks, brick_start);
        e = cudaGetLastError();
    }
    if (tmp != temp) cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "brick runs (points): %s", cudaGetErrorString(e));
    return SP_OK;
}

extern "C" int sp_brick_runs(const uint64_t* keys, int64_t n, int32_t log2_brick, int64_t* brick_start,
                             int32_t* n_bricks, void* temp, int64_t temp_bytes, void* stream) {
    if (n < 0 || n >= (1ll << 31)) return fail(SP_ERR_INVALID, "brick runs: n out of range");
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if ((n > 0 && !keys) || !brick_start || !n_bricks) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) {
        SP_CUDA(cudaMemsetAsync(n_bricks, 0, sizeof(int32_t), st));
        SP_CUDA(cudaMemsetAsync(brick_start, 0, sizeof(int64_t), st));
        return SP_OK;
    }
    const BrickHead head{keys, 3 * log2_brick};
    thrust::counting_iterator<long long> idx(0);
    size_t bytes = 0;
    SP_CUDA(cub::DeviceSelect::If(nullptr, bytes, idx, brick_start, n_bricks, (int)n, head, st));
    void* tmp = temp;
    if (!tmp || (size_t)temp_bytes < bytes) {  // no (or too small) caller scratch: stream-ordered allocation
        tmp = nullptr;
        SP_CUDA(cudaMallocAsync(&tmp, bytes, st));
    }
    const cudaError_t e = cub::DeviceSelect::If(tmp, bytes, idx, brick_start, n_bricks, (int)n, head, st);
    if (tmp != temp) cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "brick runs: %s", cudaGetErrorString(e));
    brick_runs_tail<<<1, 1, 0, st>>>(n, n_bricks, brick_start);
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

// Brick heads of sorted 32-bit keys scattered by brick id (head[b] = first index of brick b,
// -1 for empty bricks); a compaction over the brick ids then yields the runs in order
// without a pass of stream compaction over all n points.
__global__ void brick_heads32_kernel(const int32_t* __restrict__ keys, long long n, int shift, int* __restrict__ head) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int b = keys[i] >> shift;
        if (i == 0 || b != (keys[i - 1] >> shift)) head[b] = (int)i;
    }
}

struct IsHead {
    __host__ __device__ bool operator()(int v) const { return v >= 0; }
};

// morton32 keys fused with the iota of the (key, index) pairs
template <typename T>
__global__ void morton32_iota_kernel(const T* __restrict__ pts, long long n, int lo0, int lo1, int lo2, int bits,
                                     int* __restrict__ keys, int* __restrict__ iota) {
    const int hi = (1 << bits) - 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int c0 = min(max(sp::clamp_cell(pts[3 * i]) - lo0, 0), hi);
        const int c1 = min(max(sp::clamp_cell(pts[3 * i + 1]) - lo1, 0), hi);
        const int c2 = min(max(sp::clamp_cell(pts[3 * i + 2]) - lo2, 0), hi);
        keys[i] = (int)(spread3((uint32_t)c2) | (spread3((uint32_t)c1) << 1) | (spread3((uint32_t)c0) << 2));
        iota[i] = (int)i;
    }
}

// 32-bit brick heads for sp_sort_points
struct BrickHead32 {
    const int32_t* keys;
    int shift;
    __host__ __device__ bool operator()(long long i) const {
        return i == 0 || (keys[i] >> shift) != (keys[i - 1] >> shift);
    }
};

namespace {
// sp_sort_points scratch layout: keys_in | keys_out | iota | CUB scratch (sort or select)
size_t sort_points_cub_bytes(int64_t n, int end_bit) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), (int)n, 0,
                                    end_bit);
    thrust::counting_iterator<long long> idx(0);
    const BrickHead32 head{nullptr, 0};
    cub::DeviceSelect::If(nullptr, b, idx, static_cast<int64_t*>(nullptr), static_cast<int32_t*>(nullptr), (int)n, head);
    return std::max(a, b);
}
size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }
}  // namespace

extern "C" int64_t sp_sort_points_temp_bytes(int64_t n) {
    if (n <= 0 || n >= (1ll << 31)) return 0;
    return (int64_t)(3 * align256((size_t)n * 4) + sort_points_cub_bytes(n, 30));
}

// Protocol B in one sync-free call: 30-bit Morton keys of the points' unit cells relative to
// (lo0, lo1, lo2), `bits` per axis (cells clamped into [0, 2^bits) — clamping only reorders,
// any brick partition is correct), CUB radix sort of (key, index) pairs over the 3*bits key
// bits, gather of the points into key order, and the brick runs of the sorted keys
// (brick_start [n+1], count in device memory) — no host round trip.
extern "C" int sp_sort_points(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2,
                              int32_t bits, int32_t log2_brick, void* sorted_pts, int32_t* perm, int64_t* brick_start,
                              int32_t* n_bricks, void* temp, int64_t temp_bytes, void* stream) {
    if (n < 0 || n >= (1ll << 31)) return fail(SP_ERR_INVALID, "sort points: n out of range");
    if (bits < 0 || bits > 10) return fail(SP_ERR_INVALID, "bits must be in [0, 10]");
    if (log2_brick < 0 || log2_brick > bits) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (dtype != SP_F32 && dtype != SP_F64) return fail(SP_ERR_INVALID, "unknown dtype");
    if (!brick_start || !n_bricks || (n > 0 && (!pts || !perm))) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) {
        SP_CUDA(cudaMemsetAsync(n_bricks, 0, sizeof(int32_t), st));
        SP_CUDA(cudaMemsetAsync(brick_start, 0, sizeof(int64_t), st));
        return SP_OK;
    }
    const int end_bit = 3 * bits;
    const size_t seg = align256((size_t)n * 4);
    const size_t cub_bytes = sort_points_cub_bytes(n, end_bit);
    const size_t need = 3 * seg + cub_bytes;
    void* tmp = temp;
    if (!tmp || (size_t)temp_bytes < need) {
        tmp = nullptr;
        SP_CUDA(cudaMallocAsync(&tmp, need, st));
    }
    unsigned char* base = static_cast<unsigned char*>(tmp);
    int32_t* k_in = reinterpret_cast<int32_t*>(base);
    int32_t* k_out = reinterpret_cast<int32_t*>(base + seg);
    int32_t* iota = reinterpret_cast<int32_t*>(base + 2 * seg);
    void* cub_tmp = base + 3 * seg;
    cudaError_t e = cudaSuccess;
    if (dtype == SP_F32)
        morton32_iota_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, n, lo0, lo1, lo2, bits, k_in, iota);
    else
        morton32_iota_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, n, lo0, lo1, lo2, bits, k_in,
                                                                   iota);
    e = cudaGetLastError();
    size_t cb = cub_bytes;
    // The lowest end_bit % 8 key bits (the finest Morton levels inside a brick) stay unsorted
    // so that the radix sort runs whole 8-bit passes only: 27-bit keys sort in 3 passes, not 4
    // (tools/sort_bits_probe.py: -0.45 ms per 1e8 points, brick kernel unaffected).  Brick runs
    // need the brick bits sorted, so at most 3*log2_brick bits are left; SP_SORT_BEGIN_BIT
    // overrides (experiments).
    static const int begin_env = env_int("SP_SORT_BEGIN_BIT", -1);
    const int bb = std::min(begin_env >= 0 ? std::min(begin_env, 9) : end_bit % 8, 3 * log2_brick);
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(cub_tmp, cb, k_in, k_out, iota, perm, (int)n, bb, end_bit, st);
    if (e == cudaSuccess) {
        if (sorted_pts && dtype == SP_F32)
            gather_points32_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, perm, n, (float*)sorted_pts);
        else if (sorted_pts)
            gather_points32_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, perm, n, (double*)sorted_pts);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        // brick runs: scatter of the heads by brick id + compaction over the (<= n) brick ids
        // when the frame has at most n bricks (the iota segment is free after the sort), else
        // stream compaction over the n sorted keys
        const int nbf = 3 * (bits - log2_brick);
        const long long nb = 1ll << nbf;
        size_t sel = 0;
        // size query failure -> the stream-compaction path below
        const bool by_heads = nb <= n && cub::DeviceSelect::If(nullptr, sel, iota, brick_start, n_bricks, (int)nb,
                                                               IsHead{}, st) == cudaSuccess;
        if (by_heads && sel <= cub_bytes) {
            e = cudaMemsetAsync(iota, 0xff, (size_t)nb * 4, st);
            if (e == cudaSuccess) {
                brick_heads32_kernel<<<grid_for(n), 256, 0, st>>>(k_out, n, 3 * log2_brick, iota);
                e = cudaGetLastError();
            }
            cb = cub_bytes;
            if (e == cudaSuccess) e = cub::DeviceSelect::If(cub_tmp, cb, iota, brick_start, n_bricks, (int)nb, IsHead{}, st);
        } else {
            thrust::counting_iterator<long long> idx(0);
            const BrickHead32 head{k_out, 3 * log2_brick};
            cb = cub_bytes;
            e = cub::DeviceSelect::If(cub_tmp, cb, idx, brick_start, n_bricks, (int)n, head, st);
        }
    }
    if (e == cudaSuccess) {
        brick_runs_tail<<<1, 1, 0, st>>>(n, n_bricks, brick_start);
        e = cudaGetLastError();
    }
    if (tmp != temp) cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "sort points: %s", cudaGetErrorString(e));
    return SP_OK;
}

// ---------------------------------------------------------------------------------------
// Protocol B with the points as the sort payload (sp_sort_points_payload): the caller's
// points are read ONCE, coalesced, and moved through the radix sort together with their
// index, so the brick kernel afterwards reads them in brick order (no random 12/24-byte point
// reads through a permutation, which cost ~128 B of DRAM traffic per point).  Only the brick
// id is sorted (3 * (bits - log2_brick) bits: 2 onesweep passes for <= 2^16 bricks): the brick
// kernels need each brick's points contiguous, not Morton order inside the brick.
template <typename T>
struct PtIdx;  // 16 B (fp32) / 32 B (fp64) sort payload: the point and its caller index
template <>
struct __align__(16) PtIdx<float> {
    float x, y, z;
    int i;
};
template <>
struct __align__(16) PtIdx<double> {
    double x, y, z;
    long long i;
};

template <typename T>
__global__ void brick_key_payload_kernel(const T* __restrict__ pts, long long n, int lo0, int lo1, int lo2, int bits,
                                         int log2b, int* __restrict__ keys, PtIdx<T>* __restrict__ vals) {
    const int hi = (1 << bits) - 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const T x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
        const int c0 = min(max(sp::clamp_cell(x) - lo0, 0), hi) >> log2b;
        const int c1 = min(max(sp::clamp_cell(y) - lo1, 0), hi) >> log2b;
        const int c2 = min(max(sp::clamp_cell(z) - lo2, 0), hi) >> log2b;
        keys[i] = (int)(spread3((uint32_t)c2) | (spread3((uint32_t)c1) << 1) | (spread3((uint32_t)c0) << 2));
        PtIdx<T> v;
        v.x = x;
        v.y = y;
        v.z = z;
        v.i = (decltype(v.i))i;
        vals[i] = v;
    }
}

template <typename T>
__global__ void split_payload_kernel(const PtIdx<T>* __restrict__ vals, long long n, T* __restrict__ pts,
                                     int32_t* __restrict__ perm) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const PtIdx<T> v = vals[i];
        pts[3 * i] = v.x;
        pts[3 * i + 1] = v.y;
        pts[3 * i + 2] = v.z;
        perm[i] = (int32_t)v.i;
    }
}

namespace {
template <typename T>
size_t payload_cub_bytes(int64_t n, int end_bit) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<const PtIdx<T>*>(nullptr), static_cast<PtIdx<T>*>(nullptr), (int)n, 0,
                                    end_bit);
    cub::DeviceSelect::If(nullptr, b, static_cast<const int32_t*>(nullptr), static_cast<int64_t*>(nullptr),
                          static_cast<int32_t*>(nullptr), (int)std::min<int64_t>(n, 1 << 30), IsHead{});
    return std::max(a, b);
}
}  // namespace

extern "C" int64_t sp_sort_points_payload_temp_bytes(int64_t n, int32_t dtype) {
    if (n <= 0 || n >= (1ll << 31)) return 0;
    const size_t vb = dtype == SP_F64 ? sizeof(PtIdx<double>) : sizeof(PtIdx<float>);
    const size_t cub = dtype == SP_F64 ? payload_cub_bytes<double>(n, 30) : payload_cub_bytes<float>(n, 30);
    return (int64_t)(2 * align256((size_t)n * 4) + 2 * align256((size_t)n * vb) + cub);
}

extern "C" int sp_sort_points_payload(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2,
                                      int32_t bits, int32_t log2_brick, void* sorted_pts, int32_t* perm,
                                      int64_t* brick_start, int32_t* n_bricks, void* temp, int64_t temp_bytes,
                                      void* stream) {
    if (n < 0 || n >= (1ll << 31)) return fail(SP_ERR_INVALID, "sort points: n out of range");
    if (bits < 0 || bits > 10) return fail(SP_ERR_INVALID, "bits must be in [0, 10]");
    if (log2_brick < 0 || log2_brick > bits) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (dtype != SP_F32 && dtype != SP_F64) return fail(SP_ERR_INVALID, "unknown dtype");
    if (!brick_start || !n_bricks || (n > 0 && (!pts || !perm || !sorted_pts))) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) {
        SP_CUDA(cudaMemsetAsync(n_bricks, 0, sizeof(int32_t), st));
        SP_CUDA(cudaMemsetAsync(brick_start, 0, sizeof(int64_t), st));
        return SP_OK;
    }
    const int kbits = 3 * (bits - log2_brick);  // brick-id bits
    const size_t vb = dtype == SP_F64 ? sizeof(PtIdx<double>) : sizeof(PtIdx<float>);
    const size_t kseg = align256((size_t)n * 4), vseg = align256((size_t)n * vb);
    const size_t cub_bytes = dtype == SP_F64 ? payload_cub_bytes<double>(n, 30) : payload_cub_bytes<float>(n, 30);
    const size_t need = 2 * kseg + 2 * vseg + cub_bytes;
    void* tmp = temp;
    if (!tmp || (size_t)temp_bytes < need) {
        tmp = nullptr;
        SP_CUDA(cudaMallocAsync(&tmp, need, st));
    }
    unsigned char* base = static_cast<unsigned char*>(tmp);
    int32_t* k_in = reinterpret_cast<int32_t*>(base);
    int32_t* k_out = reinterpret_cast<int32_t*>(base + kseg);
    void* v_in = base + 2 * kseg;
    void* v_out = base + 2 * kseg + vseg;
    void* cub_tmp = base + 2 * kseg + 2 * vseg;
    cudaError_t e = cudaSuccess;
    size_t cb = cub_bytes;
    if (dtype == SP_F32) {
        brick_key_payload_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, n, lo0, lo1, lo2, bits, log2_brick,
                                                                     k_in, (PtIdx<float>*)v_in);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(cub_tmp, cb, k_in, k_out, (const PtIdx<float>*)v_in,
                                                (PtIdx<float>*)v_out, (int)n, 0, std::max(kbits, 1), st);
        if (e == cudaSuccess) {
            split_payload_kernel<float><<<grid_for(n), 256, 0, st>>>((const PtIdx<float>*)v_out, n, (float*)sorted_pts, perm);
            e = cudaGetLastError();
        }
    } else {
        brick_key_payload_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, n, lo0, lo1, lo2, bits,
                                                                      log2_brick, k_in, (PtIdx<double>*)v_in);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(cub_tmp, cb, k_in, k_out, (const PtIdx<double>*)v_in,
                                                (PtIdx<double>*)v_out, (int)n, 0, std::max(kbits, 1), st);
        if (e == cudaSuccess) {
            split_payload_kernel<double><<<grid_for(n), 256, 0, st>>>((const PtIdx<double>*)v_out, n, (double*)sorted_pts,
                                                                      perm);
            e = cudaGetLastError();
        }
    }
    // brick runs: the keys ARE brick ids; heads scattered by brick id (k_in is free after the
    // sort) and compacted when there are at most n bricks, else a compaction over the n keys
    if (e == cudaSuccess) {
        const long long nb = 1ll << kbits;
        size_t sel = 0;
        const bool by_heads = nb <= n && cub::DeviceSelect::If(nullptr, sel, k_in, brick_start, n_bricks, (int)nb,
                                                               IsHead{}, st) == cudaSuccess;
        if (by_heads && sel <= cub_bytes) {
            e = cudaMemsetAsync(k_in, 0xff, (size_t)nb * 4, st);
            if (e == cudaSuccess) {
                brick_heads32_kernel<<<grid_for(n), 256, 0, st>>>(k_out, n, 0, k_in);
                e = cudaGetLastError();
            }
            cb = cub_bytes;
            if (e == cudaSuccess) e = cub::DeviceSelect::If(cub_tmp, cb, k_in, brick_start, n_bricks, (int)nb, IsHead{}, st);
        } else {
            thrust::counting_iterator<long long> idx(0);
            const BrickHead32 head{k_out, 0};
            cb = cub_bytes;
            e = cub::DeviceSelect::If(cub_tmp, cb, idx, brick_start, n_bricks, (int)n, head, st);
        }
    }
    if (e == cudaSuccess) {
        brick_runs_tail<<<1, 1, 0, st>>>(n, n_bricks, brick_start);
        e = cudaGetLastError();
    }
    if (tmp != temp) cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "sort points (payload): %s", cudaGetErrorString(e));
    return SP_OK;
}

extern "C" int sp_eval_bricks_perm32(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n,
                                     int32_t dtype, const int64_t* brick_start, const int32_t* n_bricks_dev,
                                     int32_t n_bricks_cap, int32_t log2_brick, const int32_t* perm, void* out,
                                     int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0 || n_bricks_cap < 0) return fail(SP_ERR_INVALID, "negative size");
    if (n == 0 || n_bricks_cap == 0) return SP_OK;
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (!pts || !out || !brick_start || !n_bricks_dev || !perm) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        return eval_bricks_typed<float>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                        err_flag, st, n_bricks_dev, perm);
    if (dtype == SP_F64)
        return eval_bricks_typed<double>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                         err_flag, st, n_bricks_dev, perm);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

extern "C" int sp_eval_bricks_indirect(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n,
                                       int32_t dtype, const int64_t* brick_start, const int32_t* n_bricks_dev,
                                       int32_t n_bricks_cap, int32_t log2_brick, const int32_t* perm, void* out,
                                       int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0 || n_bricks_cap < 0) return fail(SP_ERR_INVALID, "negative size");
    if (n == 0 || n_bricks_cap == 0) return SP_OK;
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (!pts || !out || !brick_start || !n_bricks_dev || !perm) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        return eval_bricks_typed<float>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                        err_flag, st, n_bricks_dev, perm, perm);
    if (dtype == SP_F64)
        return eval_bricks_typed<double>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                         err_flag, st, n_bricks_dev, perm, perm);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

// Unordered protocol B: brick-order point i is pts[perm[i]], its value goes to out[i] (brick
// order, coalesced) — no scatter back to the caller's order.
extern "C" int sp_eval_bricks_unordered(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n,
                                        int32_t dtype, const int64_t* brick_start, const int32_t* n_bricks_dev,
                                        int32_t n_bricks_cap, int32_t log2_brick, const int32_t* perm, void* out,
                                        int32_t* err_flag, void* stream) {
    if (!plan) return fail(SP_ERR_INVALID, "null plan");
    int rc = check_grid(plan, grid, dtype);
    if (rc != SP_OK) return rc;
    if (n < 0 || n_bricks_cap < 0) return fail(SP_ERR_INVALID, "negative size");
    if (n == 0 || n_bricks_cap == 0) return SP_OK;
    if (log2_brick < 0 || log2_brick > 20) return fail(SP_ERR_INVALID, "log2_brick out of range");
    if (!pts || !out || !brick_start || !n_bricks_dev || !perm) return fail(SP_ERR_INVALID, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        return eval_bricks_typed<float>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                        err_flag, st, n_bricks_dev, nullptr, perm);
    if (dtype == SP_F64)
        return eval_bricks_typed<double>(plan, grid, pts, n, brick_start, n_bricks_cap, log2_brick, nullptr, out,
                                         err_flag, st, n_bricks_dev, nullptr, perm);
    return fail(SP_ERR_INVALID, "unknown dtype %d", dtype);
}

extern "C" int sp_morton_keys(const void* pts, int64_t n, int32_t dtype, uint64_t* keys, void* stream) {
    if (n <= 0) return SP_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32) morton_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, n, keys);
    else if (dtype == SP_F64) morton_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, n, keys);
    else return fail(SP_ERR_INVALID, "unknown dtype");
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

extern "C" int sp_morton_keys32(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2,
                                int32_t bits, int32_t* keys, void* stream) {
    if (n <= 0) return SP_OK;
    if (bits < 0 || bits > 10) return fail(SP_ERR_INVALID, "bits must be in [0, 10]");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32) morton32_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, n, lo0, lo1, lo2, bits, keys);
    else if (dtype == SP_F64) morton32_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, n, lo0, lo1, lo2, bits, keys);
    else return fail(SP_ERR_INVALID, "unknown dtype");
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

extern "C" int sp_scatter(const void* src, const int64_t* perm, int64_t n, int32_t dtype, void* out, void* stream) {
    if (n <= 0) return SP_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32) scatter_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)src, perm, n, (float*)out);
    else if (dtype == SP_F64) scatter_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)src, perm, n, (double*)out);
    else return fail(SP_ERR_INVALID, "unknown dtype");
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

// L2-blocked scatter out[perm[i]] = src[i] (int32 perm): destination indices are processed in
// windows of `window` elements that fit in L2, one pass over (perm, src) per window, each pass
// writing only the values whose destination falls in its window.  Every 32-byte sector of a
// window is then written completely while it is L2-resident, so it reaches HBM as one full
// sector write — a direct random scatter of 4-byte values makes HBM read-modify-write a
// sector per value (ECC granularity).  Reads (perm, src) once per window.
template <typename T>
__global__ void scatter_window_kernel(const T* __restrict__ src, const int32_t* __restrict__ perm, long long n,
                                      long long lo, long long hi, T* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long d = perm[i];
        if (d >= lo && d < hi) out[d] = src[i];
    }
}

extern "C" int sp_scatter32_blocked(const void* src, const int32_t* perm, int64_t n, int32_t dtype, int64_t window,
                                    void* out, void* stream) {
    if (n <= 0) return SP_OK;
    if (!src || !perm || !out) return fail(SP_ERR_INVALID, "null argument");
    if (dtype != SP_F32 && dtype != SP_F64) return fail(SP_ERR_INVALID, "unknown dtype");
    if (window <= 0) window = n;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (int64_t lo = 0; lo < n; lo += window) {
        const int64_t hi = std::min<int64_t>(n, lo + window);
        if (dtype == SP_F32)
            scatter_window_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)src, perm, n, lo, hi, (float*)out);
        else
            scatter_window_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)src, perm, n, lo, hi, (double*)out);
        SP_CUDA(cudaGetLastError());
    }
    return SP_OK;
}

// Result scatter for a permutation, without partial-sector writes: a radix sort of the
// (destination, value) pairs by the destination's high bits only (bits >= kPermWinBits, two
// 8-bit onesweep passes at 1e8) puts the 2^kPermWinBits values of every destination window
// into that window's own slot range (perm is a permutation, so each window holds exactly
// its size); one CTA per window then places them in shared memory and writes the window
// with full coalesced stores.
constexpr int kPermWinBits = 11;

template <typename T>
__global__ void __launch_bounds__(256) perm_window_kernel(const int32_t* __restrict__ dst, const T* __restrict__ val,
                                                          long long n, T* __restrict__ out) {
    constexpr int W = 1 << kPermWinBits;
    __shared__ T buf[W];
    for (long long w = blockIdx.x; w * W < n; w += gridDim.x) {
        const long long b0 = w * W;
        const int m = (int)std::min<long long>(W, n - b0);
        for (int i = threadIdx.x; i < m; i += 256) buf[dst[b0 + i] & (W - 1)] = val[b0 + i];
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += 256) out[b0 + i] = buf[i];
        __syncthreads();
    }
}

namespace {
template <typename T>
size_t perm_scatter_cub_bytes(int64_t n) {
    size_t a = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<const T*>(nullptr), static_cast<T*>(nullptr), (int)n, kPermWinBits, 31);
    return a;
}
int perm_end_bit(int64_t n) {
    int b = 1;
    while (b < 31 && (1ll << b) < n) ++b;
    return std::max(b, kPermWinBits + 1);
}
}  // namespace

extern "C" int64_t sp_scatter32_perm_temp_bytes(int64_t n, int32_t dtype) {
    if (n <= 0 || n >= (1ll << 31)) return 0;
    const size_t e = dtype == SP_F64 ? 8 : 4;
    const size_t cub = dtype == SP_F64 ? perm_scatter_cub_bytes<double>(n) : perm_scatter_cub_bytes<float>(n);
    return (int64_t)(align256((size_t)n * 4) + align256((size_t)n * e) + cub);
}

extern "C" int sp_scatter32_perm(const void* src, const int32_t* perm, int64_t n, int32_t dtype, void* out, void* temp,
                                 int64_t temp_bytes, void* stream) {
    if (n <= 0) return SP_OK;
    if (n >= (1ll << 31)) return fail(SP_ERR_INVALID, "permutation scatter: n out of range");
    if (!src || !perm || !out) return fail(SP_ERR_INVALID, "null argument");
    if (dtype != SP_F32 && dtype != SP_F64) return fail(SP_ERR_INVALID, "unknown dtype");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t e = dtype == SP_F64 ? 8 : 4;
    const size_t ds = align256((size_t)n * 4), vs = align256((size_t)n * e);
    const size_t need = (size_t)sp_scatter32_perm_temp_bytes(n, dtype);
    void* tmp = temp;
    if (!tmp || (size_t)temp_bytes < need) {
        tmp = nullptr;
        SP_CUDA(cudaMallocAsync(&tmp, need, st));
    }
    unsigned char* base = static_cast<unsigned char*>(tmp);
    int32_t* dsorted = reinterpret_cast<int32_t*>(base);
    void* vsorted = base + ds;
    void* cub_tmp = base + ds + vs;
    size_t cb = need - ds - vs;
    const int end_bit = perm_end_bit(n);
    const long long nwin = (n + (1 << kPermWinBits) - 1) >> kPermWinBits;
    const int blocks = (int)std::min<long long>(nwin, 148ll * 8);
    cudaError_t err;
    if (dtype == SP_F32) {
        err = cub::DeviceRadixSort::SortPairs(cub_tmp, cb, perm, dsorted, (const float*)src, (float*)vsorted, (int)n,
                                              kPermWinBits, end_bit, st);
        if (err == cudaSuccess) {
            perm_window_kernel<float><<<blocks, 256, 0, st>>>(dsorted, (const float*)vsorted, n, (float*)out);
            err = cudaGetLastError();
        }
    } else {
        err = cub::DeviceRadixSort::SortPairs(cub_tmp, cb, perm, dsorted, (const double*)src, (double*)vsorted, (int)n,
                                              kPermWinBits, end_bit, st);
        if (err == cudaSuccess) {
            perm_window_kernel<double><<<blocks, 256, 0, st>>>(dsorted, (const double*)vsorted, n, (double*)out);
            err = cudaGetLastError();
        }
    }
    if (tmp != temp) cudaFreeAsync(tmp, st);
    if (err != cudaSuccess) return fail(SP_ERR_CUDA, "permutation scatter: %s", cudaGetErrorString(err));
    return SP_OK;
}

extern "C" int sp_gather_points(const void* pts, const int64_t* perm, int64_t n, int32_t dtype, void* dst, void* stream) {
    if (n <= 0) return SP_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32) gather_points_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)pts, perm, n, (float*)dst);
    else if (dtype == SP_F64) gather_points_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)pts, perm, n, (double*)dst);
    else return fail(SP_ERR_INVALID, "unknown dtype");
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}
