// h2_file.cpp -- the library's reader of the .h2m flat file (include/h2.h h2_file_info,
// h2_create_from_file).  Layout: SPEC.md:156 ("header {N, m, depth, level ranks}, then
// level-ordered arrays"), a 512-byte little-endian header and 64-byte-aligned sections in the
// order documented in include/h2.h.  Each rank reads only the byte ranges of its own view
// (its branch at levels >= C = log2 P, the top levels replicated) and hands them
// to h2_create as host arrays.
#include "../../include/h2.h"
#include "h2_internal.h"

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

struct FileHeader {
    uint32_t version, dtype, dim, m, q, flags, kernel_id, reserved;
    uint64_t N, n_D, seed;
    double eta, kpar[4];
    int32_t k[32];
    int64_t nS[32];
};

int ferr(int code, const std::string &m)
{
    h2::set_last_error(m);
    return code;
}

struct File {
    FILE *f = nullptr;
    FileHeader h{};
    size_t esz = 8;
    ~File() { if (f) fclose(f); }
    int open(const char *path)
    {
        if (!path) return ferr(H2_ERR_ARG, "path is NULL");
        f = fopen(path, "rb");
        if (!f) return ferr(H2_ERR_ARG, std::string("cannot open ") + path);
        unsigned char hdr[512];
        if (fread(hdr, 1, 512, f) != 512) return ferr(H2_ERR_STRUCT, ".h2m header truncated");
        if (memcmp(hdr, "H2MFLAT1", 8) != 0) return ferr(H2_ERR_STRUCT, "not an .h2m file (magic)");
        memcpy(&h.version, hdr + 8, 32);
        memcpy(&h.N, hdr + 40, 24);
        memcpy(&h.eta, hdr + 64, 40);
        memcpy(h.k, hdr + 128, 128);
        memcpy(h.nS, hdr + 256, 256);
        if (h.version != 1) return ferr(H2_ERR_STRUCT, "unsupported .h2m version");
        if (h.dtype > 1) return ferr(H2_ERR_STRUCT, "bad dtype in .h2m header");
        if (h.q > 30 || h.m < 1 || h.dim < 1) return ferr(H2_ERR_STRUCT, "bad sizes in .h2m header");
        esz = h.dtype == 0 ? 8 : 4;
        return H2_OK;
    }
};

// Byte offsets of every section (sequential, each 64-byte aligned), from the header alone.
struct Sections {
    int64_t points, perm, leaf_ptr, U, V;
    std::vector<int64_t> E, F, Srp, Scol, S;
    int64_t Drp, Dcol, D, end;
};

Sections sections(const FileHeader &h, size_t esz)
{
    Sections s;
    int64_t pos = 512;
    auto sec = [&](int64_t bytes) {
        pos = (pos + 63) / 64 * 64;
        int64_t at = pos;
        pos += bytes;
        return at;
    };
    const int q = (int)h.q;
    const int64_t nleaf = (int64_t)1 << q;
    s.points = sec((int64_t)h.N * h.dim * 8);
    s.perm = sec((int64_t)h.N * 8);
    s.leaf_ptr = sec((nleaf + 1) * 8);
    s.U = sec(nleaf * h.k[q] * (int64_t)h.m * esz);
    s.V = (h.flags & 1) ? s.U : sec(nleaf * h.k[q] * (int64_t)h.m * esz);
    s.E.assign(q + 1, -1);
    s.F.assign(q + 1, -1);
    for (int l = 1; l <= q; ++l) s.E[l] = sec(((int64_t)1 << l) * h.k[l] * h.k[l - 1] * (int64_t)esz);
    for (int l = 1; l <= q; ++l)
        s.F[l] = (h.flags & 2) ? s.E[l] : sec(((int64_t)1 << l) * h.k[l] * h.k[l - 1] * (int64_t)esz);
    s.Srp.assign(q + 1, 0);
    s.Scol.assign(q + 1, 0);
    s.S.assign(q + 1, 0);
    for (int l = 0; l <= q; ++l) {
        s.Srp[l] = sec((((int64_t)1 << l) + 1) * 8);
        s.Scol[l] = sec(h.nS[l] * 4);
        s.S[l] = sec(h.nS[l] * h.k[l] * (int64_t)h.k[l] * esz);
    }
    s.Drp = sec((nleaf + 1) * 8);
    s.Dcol = sec((int64_t)h.n_D * 4);
    s.D = sec((int64_t)h.n_D * h.m * (int64_t)h.m * esz);
    s.end = pos;
    return s;
}

template <typename V>
int read_at(FILE *f, int64_t off, int64_t count, V &out)
{
    out.resize((size_t)count);
    if (count == 0) return H2_OK;
    if (fseeko(f, (off_t)off, SEEK_SET) != 0) return ferr(H2_ERR_STRUCT, ".h2m seek failed");
    if (fread(out.data(), sizeof(out[0]), (size_t)count, f) != (size_t)count) return ferr(H2_ERR_STRUCT, ".h2m file truncated");
    return H2_OK;
}

int read_bytes(FILE *f, int64_t off, int64_t bytes, std::vector<unsigned char> &out)
{
    return read_at(f, off, bytes, out);
}

}  // namespace

extern "C" int h2_file_info(const char *path, int64_t info[8])
{
    if (!info) return ferr(H2_ERR_ARG, "info is NULL");
    File fl;
    int rc = fl.open(path);
    if (rc != H2_OK) return rc;
    int64_t nS = 0;
    for (uint32_t l = 0; l <= fl.h.q; ++l) nS += fl.h.nS[l];
    int64_t v[8] = {(int64_t)fl.h.N, (int64_t)fl.h.dim, (int64_t)fl.h.m, (int64_t)fl.h.q,
                    (int64_t)fl.h.dtype, nS, (int64_t)fl.h.n_D, (int64_t)fl.h.k[fl.h.q]};
    memcpy(info, v, sizeof(v));
    Sections s = sections(fl.h, fl.esz);
    if (fseeko(fl.f, 0, SEEK_END) != 0 || (int64_t)ftello(fl.f) < s.end)
        return ferr(H2_ERR_STRUCT, ".h2m file shorter than its header says");
    return H2_OK;
}

namespace {

// One rank's view read from the file: owning buffers plus the h2_desc pointing into them.
struct View {
    std::vector<int64_t> leaf_ptr, drp;
    std::vector<unsigned char> U, V, D;
    std::vector<std::vector<unsigned char>> E, F, S;
    std::vector<std::vector<int64_t>> Srp;
    std::vector<std::vector<int32_t>> Scol;
    std::vector<int32_t> dcol, kk;
    std::vector<const void *> Ep, Fp, Sp;
    std::vector<const int64_t *> Srpp;
    std::vector<const int32_t *> Scolp;
    h2_desc d{};
};

int load_view(const char *path, int rank, int nranks, View &v)
{
    File fl;
    int rc = fl.open(path);
    if (rc != H2_OK) return rc;
    const FileHeader &h = fl.h;
    const int q = (int)h.q;
    if (nranks < 1 || (nranks & (nranks - 1))) return ferr(H2_ERR_STRUCT, "nranks must be a power of two");
    if (rank < 0 || rank >= nranks) return ferr(H2_ERR_ARG, "rank out of range");
    int C = 0;
    while ((1 << C) < nranks) ++C;
    if (C > q) return ferr(H2_ERR_STRUCT, "P too large for depth (P > 2^q)");
    Sections s = sections(h, fl.esz);
    auto held = [&](int l, int64_t &a, int64_t &b) {
        if (l < C) { a = 0; b = (int64_t)1 << l; }
        else { int64_t w = (int64_t)1 << (l - C); a = rank * w; b = a + w; }
    };
    const size_t esz = fl.esz;
    int64_t la, lb;
    held(q, la, lb);
    std::vector<int64_t> lp_all;
    if ((rc = read_at(fl.f, s.leaf_ptr + la * 8, lb - la + 1, lp_all)) != H2_OK) return rc;
    const int64_t r0 = lp_all[0];
    v.leaf_ptr.resize(lp_all.size());
    for (size_t i = 0; i < lp_all.size(); ++i) v.leaf_ptr[i] = lp_all[i] - r0;
    const int64_t ub = (int64_t)h.k[q] * h.m * esz;
    if ((rc = read_bytes(fl.f, s.U + la * ub, (lb - la) * ub, v.U)) != H2_OK) return rc;
    if (!(h.flags & 1) && (rc = read_bytes(fl.f, s.V + la * ub, (lb - la) * ub, v.V)) != H2_OK) return rc;
    v.E.assign(q + 1, {});
    v.F.assign(q + 1, {});
    v.S.assign(q + 1, {});
    v.Srp.assign(q + 1, {});
    v.Scol.assign(q + 1, {});
    for (int l = 0; l <= q; ++l) {
        int64_t a, b;
        held(l, a, b);
        if (l >= 1) {
            const int64_t eb = (int64_t)h.k[l] * h.k[l - 1] * esz;
            if ((rc = read_bytes(fl.f, s.E[l] + a * eb, (b - a) * eb, v.E[l])) != H2_OK) return rc;
            if (!(h.flags & 2) && (rc = read_bytes(fl.f, s.F[l] + a * eb, (b - a) * eb, v.F[l])) != H2_OK) return rc;
        }
        std::vector<int64_t> rp;
        if ((rc = read_at(fl.f, s.Srp[l] + a * 8, b - a + 1, rp)) != H2_OK) return rc;
        const int64_t b0 = rp[0], b1 = rp.back();
        if (b0 < 0 || b1 < b0 || b1 > h.nS[l]) return ferr(H2_ERR_STRUCT, ".h2m S_rowptr out of range");
        for (auto &x : rp) x -= b0;
        v.Srp[l] = rp;
        if ((rc = read_at(fl.f, s.Scol[l] + b0 * 4, b1 - b0, v.Scol[l])) != H2_OK) return rc;
        const int64_t sb = (int64_t)h.k[l] * h.k[l] * esz;
        if ((rc = read_bytes(fl.f, s.S[l] + b0 * sb, (b1 - b0) * sb, v.S[l])) != H2_OK) return rc;
    }
    if ((rc = read_at(fl.f, s.Drp + la * 8, lb - la + 1, v.drp)) != H2_OK) return rc;
    const int64_t d0 = v.drp[0], d1 = v.drp.back();
    if (d0 < 0 || d1 < d0 || d1 > (int64_t)h.n_D) return ferr(H2_ERR_STRUCT, ".h2m D_rowptr out of range");
    for (auto &x : v.drp) x -= d0;
    if ((rc = read_at(fl.f, s.Dcol + d0 * 4, d1 - d0, v.dcol)) != H2_OK) return rc;
    const int64_t db = (int64_t)h.m * h.m * esz;
    if ((rc = read_bytes(fl.f, s.D + d0 * db, (d1 - d0) * db, v.D)) != H2_OK) return rc;
    // the h2_desc (host arrays, copied by h2_create)
    v.Ep.assign(q + 1, nullptr);
    v.Fp.assign(q + 1, nullptr);
    v.Sp.assign(q + 1, nullptr);
    v.Srpp.assign(q + 1, nullptr);
    v.Scolp.assign(q + 1, nullptr);
    for (int l = 0; l <= q; ++l) {
        if (l >= 1) { v.Ep[l] = v.E[l].data(); v.Fp[l] = (h.flags & 2) ? v.E[l].data() : v.F[l].data(); }
        v.Sp[l] = v.S[l].empty() ? nullptr : v.S[l].data();
        v.Srpp[l] = v.Srp[l].data();
        v.Scolp[l] = v.Scol[l].data();
    }
    v.kk.assign(h.k, h.k + q + 1);
    h2_desc &d = v.d;
    d.dtype = h.dtype == 0 ? H2_F64 : H2_F32;
    d.mem = H2_MEM_HOST;
    d.depth = q;
    d.leaf_size = (int32_t)h.m;
    d.rank = rank;
    d.nranks = nranks;
    d.n_local = v.leaf_ptr.back();
    d.level_rank = v.kk.data();
    d.leaf_ptr = v.leaf_ptr.data();
    d.U_leaf = v.U.data();
    d.V_leaf = (h.flags & 1) ? v.U.data() : v.V.data();
    d.E = v.Ep.data();
    d.F = v.Fp.data();
    d.S_rowptr = v.Srpp.data();
    d.S_col = v.Scolp.data();
    d.S = v.Sp.data();
    d.D_rowptr = v.drp.data();
    d.D_col = v.dcol.empty() ? nullptr : v.dcol.data();
    d.D = v.D.empty() ? nullptr : v.D.data();
    return H2_OK;
}

}  // namespace

extern "C" int h2_create_from_file(const char *path, int rank, int nranks, int nv_max, const void *nccl_unique_id,
                                   h2_handle *out)
{
    if (!out) return ferr(H2_ERR_ARG, "out is NULL");
    *out = nullptr;
    try {
        View v;
        int rc = load_view(path, rank, nranks, v);
        if (rc != H2_OK) return rc;
        return h2_create(&v.d, nv_max, nccl_unique_id, out);
    } catch (const std::exception &e) {
        return ferr(H2_ERR_OOM, std::string("h2_create_from_file: ") + e.what());
    }
}

extern "C" int h2_group_create_from_file(const char *path, int P, int nv_max, h2_handle *out)
{
    if (!out || P < 1) return ferr(H2_ERR_ARG, "bad argument");
    try {
        std::vector<View> views(P);
        std::vector<const h2_desc *> descs(P);
        for (int o = 0; o < P; ++o) {
            int rc = load_view(path, o, P, views[o]);
            if (rc != H2_OK) return rc;
            descs[o] = &views[o].d;
        }
        return h2_group_create(descs.data(), P, nv_max, out);
    } catch (const std::exception &e) {
        return ferr(H2_ERR_OOM, std::string("h2_group_create_from_file: ") + e.what());
    }
}
