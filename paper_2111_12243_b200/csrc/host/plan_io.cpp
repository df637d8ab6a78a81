// Binary plan files: the reference can only write a
// JSON dump (plan_io.cpp:52-83), GB-scale at configs 3/5 and not reloadable.
// This format stores the structure-of-arrays plan as it is held in memory --
// compact codelet records for mined plans, explicit descriptors for imported
// ones -- so a plan inspected once is reloaded without re-inspection.
//
// Layout (little-endian): "PSCPLAN\0", u32 version, the scalar fields, then
// every array as u64 element count + raw elements, in a fixed order.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_types.hpp"
#include "common.hpp"

namespace pscb {
namespace {

constexpr char kMagic[8] = {'P', 'S', 'C', 'P', 'L', 'A', 'N', '\0'};
constexpr uint32_t kVersion = 2;  // 2: + the structure hash of the matrix a mined plan came from

struct File {
    std::FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

template <class T>
void put(std::FILE* f, const T& v) {
    require(std::fwrite(&v, sizeof(T), 1, f) == 1, "plan_save: write failed");
}
template <class T>
void put_vec(std::FILE* f, const std::vector<T>& v) {
    put<uint64_t>(f, v.size());
    if (!v.empty()) require(std::fwrite(v.data(), sizeof(T), v.size(), f) == v.size(), "plan_save: write failed");
}
template <class T>
T get(std::FILE* f) {
    T v{};
    require(std::fread(&v, sizeof(T), 1, f) == 1, "plan_load: truncated file");
    return v;
}
template <class T>
void get_vec(std::FILE* f, std::vector<T>& v) {
    const uint64_t n = get<uint64_t>(f);
    require(n < (uint64_t{1} << 40), "plan_load: corrupt array length");
    v.resize(n);
    if (n) require(std::fread(v.data(), sizeof(T), n, f) == n, "plan_load: truncated file");
}

template <class F>
void arrays(Plan& p, F&& f) {  // the fixed order of the arrays
    f(p.part_group_ptr);
    f(p.g_row_begin);
    f(p.g_row_end);
    f(p.g_strategy);
    f(p.g_cost);
    f(p.g_codelet_ptr);
    f(p.c_kind);
    f(p.c_m);
    f(p.c_n);
    f(p.c_row);
    f(p.c_mat_base);
    f(p.c_mat_so);
    f(p.c_vec_base);
    f(p.c_vec_so);
    f(p.d_form);
    f(p.d_base);
    f(p.d_so);
    f(p.d_si);
    f(p.d_tab_ptr);
    f(p.tables);
    f(p.g_fin_ptr);
    f(p.f_row);
    f(p.f_diag);
    f(p.f_rhs);
}

}  // namespace

void plan_save(const Plan& plan, const std::string& path) {
    File file;
    file.f = std::fopen(path.c_str(), "wb");
    require(file.f != nullptr, "plan_save: cannot open " + path);
    std::FILE* f = file.f;
    require(std::fwrite(kMagic, 1, 8, f) == 8, "plan_save: write failed");
    put(f, kVersion);
    put(f, plan.kernel);
    put(f, plan.n_rows);
    put(f, plan.n_cols);
    put(f, plan.nnz);
    put(f, plan.window);
    put(f, plan.target_groups);
    put<uint8_t>(f, plan.mined ? 1 : 0);
    put<uint64_t>(f, plan.structure);
    Plan& p = const_cast<Plan&>(plan);
    arrays(p, [&](auto& v) { put_vec(f, v); });
    require(std::fflush(f) == 0, "plan_save: write failed");
}

Plan plan_load(const std::string& path) {
    File file;
    file.f = std::fopen(path.c_str(), "rb");
    require(file.f != nullptr, "plan_load: cannot open " + path);
    std::FILE* f = file.f;
    char magic[8];
    require(std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kMagic, 8) == 0, "plan_load: not a plan file");
    const uint32_t version = get<uint32_t>(f);
    require(version == 1 || version == kVersion, "plan_load: unsupported version");
    Plan p;
    p.kernel = get<int32_t>(f);
    p.n_rows = get<int32_t>(f);
    p.n_cols = get<int32_t>(f);
    p.nnz = get<int64_t>(f);
    p.window = get<int32_t>(f);
    p.target_groups = get<int32_t>(f);
    p.mined = get<uint8_t>(f) != 0;
    if (version >= 2) p.structure = get<uint64_t>(f);
    arrays(p, [&](auto& v) { get_vec(f, v); });
    // structural sanity (binding checks the matrix: the structure hash, or
    // validate_plan for a version-1 file)
    require(p.kernel == PSC_KERNEL_SPMV || p.kernel == PSC_KERNEL_SPTRSV, "plan_load: bad kernel");
    const int64_t ng = p.n_groups(), nc = p.n_codelets();
    require(!p.part_group_ptr.empty() && p.part_group_ptr.back() == ng, "plan_load: inconsistent partitions");
    require(static_cast<int64_t>(p.g_row_end.size()) == ng && static_cast<int64_t>(p.g_strategy.size()) == ng &&
                static_cast<int64_t>(p.g_cost.size()) == ng && static_cast<int64_t>(p.g_codelet_ptr.size()) == ng + 1 &&
                p.g_codelet_ptr.back() == nc,
            "plan_load: inconsistent groups");
    require(static_cast<int64_t>(p.c_m.size()) == nc && static_cast<int64_t>(p.c_n.size()) == nc,
            "plan_load: inconsistent codelets");
    if (p.mined) {
        require(static_cast<int64_t>(p.c_row.size()) == nc && static_cast<int64_t>(p.c_vec_so.size()) == nc,
                "plan_load: inconsistent codelet records");
    } else {
        require(static_cast<int64_t>(p.d_form.size()) == 3 * nc && static_cast<int64_t>(p.d_tab_ptr.size()) == 3 * nc + 1,
                "plan_load: inconsistent descriptors");
    }
    return p;
}

}  // namespace pscb

using namespace pscb;

PSC_API psc_status psc_plan_save(const psc_plan* plan, const char* path) {
    return guarded([&] {
        require(plan && path, "psc_plan_save: null argument");
        plan_save(plan->p, path);
    });
}

PSC_API psc_status psc_plan_load(const char* path, psc_plan** out) {
    return guarded([&] {
        require(path && out, "psc_plan_load: null argument");
        *out = new psc_plan(plan_load(path));
    });
}
