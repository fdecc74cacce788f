// The .apr container (docs/FORMATS.md; io.hpp:102-183) read straight into a
// device handle and written back from one, byte for byte as the reference's
// write_apr does: magic "APRB", version 1, source dims (u32 x 3), BuildParams,
// the leaf and interior access blocks, the leaf values.  Little-endian host
// assumed (x86-64 / aarch64), as the format is.
//
// The reader applies the reference reader's checks in its order with its
// messages (read_pod / read_array / read_access / read_apr), then validate --
// on the device (aprgpu_validate_access), not over the pixels.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.cuh"

namespace aprgpu {
namespace {

struct IoFail {
    int status;
    std::string msg;
};
[[noreturn]] void bad(const std::string& m) { throw IoFail{APRGPU_ERR_BAD_FORMAT, m}; }

struct Reader {
    FILE* f;
    template <typename T>
    T pod(const char* field) {
        T v{};
        if (std::fread(&v, sizeof(T), 1, f) != 1)
            throw IoFail{APRGPU_ERR_TRUNCATED, std::string("unexpected end of file reading ") + field};
        return v;
    }
    template <typename T>
    std::vector<T> array(const char* field, uint64_t max_count) {
        const uint64_t n = pod<uint64_t>(field);
        if (n > max_count) bad(std::string("implausible element count for ") + field);
        std::vector<T> v(n);
        if (n && std::fread(v.data(), sizeof(T), n, f) != n)
            throw IoFail{APRGPU_ERR_TRUNCATED, std::string("unexpected end of file reading ") + field};
        return v;
    }
};

struct HostAccess {
    int l_min = 0, l_max = 0;
    std::vector<int32_t> zd, xd, yd;
    std::vector<uint64_t> level_offset, xz_end;
    std::vector<uint16_t> y;
    aprgpu_access_desc desc() const {
        aprgpu_access_desc d{};
        d.l_min = l_min;
        d.l_max = l_max;
        d.z_dim = zd.data();
        d.x_dim = xd.data();
        d.y_dim = yd.data();
        d.y_idx = y.empty() ? nullptr : y.data();
        d.n_particles = y.size();
        d.xz_end = xz_end.empty() ? nullptr : xz_end.data();
        d.n_rows = xz_end.size();
        d.level_offset = level_offset.data();
        return d;
    }
};

HostAccess read_access(Reader& r, const std::string& what) {  // io.hpp:80-100
    HostAccess a;
    a.l_min = r.pod<int32_t>("l_min");
    a.l_max = r.pod<int32_t>("l_max");
    if (a.l_min < 0 || a.l_max < a.l_min || a.l_max > 40) bad(what + ": bad level range");
    for (int l = 0; l <= a.l_max; ++l) {
        a.zd.push_back(r.pod<int32_t>("z_dim"));
        a.xd.push_back(r.pod<int32_t>("x_dim"));
        a.yd.push_back(r.pod<int32_t>("y_dim"));
        if (a.zd.back() < 0 || a.xd.back() < 0 || a.yd.back() < 0 || a.yd.back() > 65536)
            bad(what + ": bad level grid dims");
    }
    const uint64_t cap = uint64_t(1) << 40;
    a.level_offset = r.array<uint64_t>("level_offset", cap);
    a.xz_end = r.array<uint64_t>("xz_end", cap);
    a.y = r.array<uint16_t>("y_idx", cap);
    if (a.level_offset.size() != static_cast<size_t>(a.l_max + 1)) bad(what + ": level_offset length mismatch");
    return a;
}

struct Writer {
    FILE* f;
    bool ok = true;
    template <typename T>
    void pod(T v) {
        ok = ok && std::fwrite(&v, sizeof(T), 1, f) == 1;
    }
    template <typename T>
    void array(const T* p, uint64_t n) {
        pod<uint64_t>(n);
        if (n) ok = ok && std::fwrite(p, sizeof(T), n, f) == n;
    }
};

void write_access(Writer& w, const aprgpu_apr* apr, int which) {  // io.hpp:66-77
    const DevAccess& a = which == APRGPU_LEAF ? apr->leaf : apr->tree;
    aprgpu_access_info info{};
    aprgpu_access_get_info(apr, which, &info);
    const size_t n = static_cast<size_t>(a.l_max) + 1;
    std::vector<uint16_t> y(a.n_particles);
    std::vector<uint64_t> xz(a.n_rows), lo(n);
    std::vector<int32_t> zd(n), xd(n), yd(n);
    if (aprgpu_download_access(apr, which, y.data(), xz.data(), lo.data(), zd.data(), xd.data(), yd.data()) !=
        APRGPU_OK)
        fail(APRGPU_ERR_CUDA, aprgpu_last_error());
    w.pod<int32_t>(a.l_min);
    w.pod<int32_t>(a.l_max);
    for (size_t l = 0; l < n; ++l) {
        w.pod<int32_t>(zd[l]);
        w.pod<int32_t>(xd[l]);
        w.pod<int32_t>(yd[l]);
    }
    w.array(lo.data(), lo.size());
    w.array(xz.data(), xz.size());
    w.array(y.data(), y.size());
}

}  // namespace

// read_apr (io.hpp:131-169) into a device handle; returns a status, message in msg
int load_apr_host(aprgpu_ctx* ctx, const char* path, aprgpu_apr** out, std::string& msg) {
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), std::fclose);
    if (!f) {
        msg = std::string("cannot open for reading: ") + path;
        return APRGPU_ERR_IO;
    }
    try {
        Reader r{f.get()};
        char magic[4];
        if (std::fread(magic, 1, 4, r.f) != 4) throw IoFail{APRGPU_ERR_TRUNCATED, "unexpected end of file reading magic"};
        if (std::memcmp(magic, "APRB", 4) != 0) bad("not an APR file (bad magic)");
        const uint8_t version = r.pod<uint8_t>("version");
        if (version != 1) bad("unsupported APR file version " + std::to_string(version));
        int32_t dims[3];
        for (int d = 0; d < 3; ++d) {
            const uint32_t v = r.pod<uint32_t>("dims");
            if (v == 0 || v > (1u << 30)) bad("bad source dims");
            dims[d] = static_cast<int32_t>(v);
        }
        aprgpu_build_params p{};
        p.rel_error = r.pod<double>("rel_error");
        const uint8_t smode = r.pod<uint8_t>("sigma mode");
        if (smode > 1) bad("bad sigma mode");
        p.sigma_mode = smode;
        p.sigma_value = r.pod<double>("sigma value");
        p.sigma_window = r.pod<int32_t>("sigma window");
        p.sigma_floor = r.pod<double>("sigma floor");
        const uint8_t gmode = r.pod<uint8_t>("gradient mode");
        if (gmode > 1) bad("bad gradient mode");
        p.gradient_mode = gmode;
        p.smoothing_passes = r.pod<int32_t>("smoothing passes");
        const HostAccess leaf = read_access(r, "leaf access");
        const HostAccess tree = read_access(r, "tree access");
        const std::vector<float> values = r.array<float>("leaf values", uint64_t(1) << 40);
        if (values.size() != leaf.y.size()) bad("leaf value count does not match particle count");
        const aprgpu_access_desc ld = leaf.desc(), td = tree.desc();
        int ok = 0;
        char vmsg[512];
        int st = aprgpu_validate_access(ctx, &ld, dims, &ok, vmsg, sizeof(vmsg));
        if (st != APRGPU_OK) {
            msg = aprgpu_last_error();
            return st;
        }
        if (!ok) bad(std::string("invalid APR structure: ") + vmsg);
        aprgpu_apr* apr = nullptr;
        st = aprgpu_upload_access(ctx, &ld, &td, dims, &apr);
        if (st != APRGPU_OK) {
            msg = aprgpu_last_error();
            return st;
        }
        apr->params = p;
        apr->built_values.ensure(4 * values.size() + 4);
        if (!values.empty()) {
            const cudaError_t e = cudaMemcpy(apr->built_values.p, values.data(), 4 * values.size(), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                aprgpu_apr_free(apr);
                msg = cudaGetErrorString(e);
                return APRGPU_ERR_CUDA;
            }
        }
        *out = apr;
        return APRGPU_OK;
    } catch (const IoFail& e) {
        msg = e.msg;
        return e.status;
    }
}

// write_apr (io.hpp:104-126); values on the host
int save_apr_host(const aprgpu_apr* apr, const char* path, const float* values, std::string& msg) {
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), std::fclose);
    if (!f) {
        msg = std::string("cannot open for writing: ") + path;
        return APRGPU_ERR_IO;
    }
    Writer w{f.get()};
    std::fwrite("APRB", 1, 4, w.f);
    w.pod<uint8_t>(1);
    for (int d = 0; d < 3; ++d) w.pod<uint32_t>(static_cast<uint32_t>(apr->dims[d]));
    const aprgpu_build_params& p = apr->params;
    w.pod<double>(p.rel_error);
    w.pod<uint8_t>(static_cast<uint8_t>(p.sigma_mode));
    w.pod<double>(p.sigma_value);
    w.pod<int32_t>(p.sigma_window);
    w.pod<double>(p.sigma_floor);
    w.pod<uint8_t>(static_cast<uint8_t>(p.gradient_mode));
    w.pod<int32_t>(p.smoothing_passes);
    write_access(w, apr, APRGPU_LEAF);
    write_access(w, apr, APRGPU_TREE);
    w.array(values, apr->leaf.n_particles);
    if (!w.ok || std::fflush(w.f) != 0) {
        msg = std::string("write failed: ") + path;
        return APRGPU_ERR_IO;
    }
    return APRGPU_OK;
}

}  // namespace aprgpu
