// xa_image_io.cpp — image file I/O of the reference's evaluation harness
// (SURVEY.md §8(f) row 4): load_image / save_image / save_png_rgb
// (proj/include/xaffine/image_io.hpp:14-24, proj/src/image_io.cpp).
//
// Host code (no device work): PNM (P2/P3/P5/P6, '#' comments, maxval <= 255)
// and PNG read as grayscale with the reference's luminance
// (float)(0.299 R + 0.587 G + 0.114 B) in double (image_io.cpp:23-25); 8-bit
// grayscale PGM / PNG written with the reference's quantisation lround + clamp
// to [0, 255] (image_io.cpp:18-21), which is also the rule the device applies
// to uint8 views. PNG goes through zlib directly (libpng is absent in this
// image): the decoder applies the transforms the reference requests from
// libpng -- 16-bit samples keep their high byte (png_set_strip_16), palettes
// expand to RGB, 1/2/4-bit gray scales to 8 bits, alpha is dropped, Adam7
// interlacing is undone (png_read_image) -- so the decoded pixels equal the
// reference's. The encoder writes one IDAT of filter-0 rows.
#include <zlib.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/xaffine_b200.h"

namespace xa {
int host_error(int code, const std::string& msg);
}

namespace {

struct IoFail {
    std::string msg;
};

uint8_t quantize(float v) {  // image_io.cpp:18-21
    const long q = std::lround(v);
    return static_cast<uint8_t>(std::min<long>(std::max<long>(q, 0), 255));
}

float luminance(double r, double g, double b) { return static_cast<float>(0.299 * r + 0.587 * g + 0.114 * b); }

bool has_suffix(const std::string& s, const std::string& suf) {
    if (s.size() < suf.size()) return false;
    std::string tail = s.substr(s.size() - suf.size());
    for (char& c : tail) c = (char)std::tolower((unsigned char)c);
    return tail == suf;
}

std::vector<uint8_t> read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoFail{"cannot open image: " + path};
    return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

// ------------------------------------------------------------------ PNM

struct Cursor {
    const std::vector<uint8_t>& b;
    size_t i = 0;
    int peek() const { return i < b.size() ? b[i] : EOF; }
};

// whitespace and '#' comment lines, then a decimal integer (image_io.cpp:35-52)
int next_pnm_int(Cursor& c) {
    while (true) {
        const int ch = c.peek();
        if (ch == EOF) throw IoFail{"unexpected end of PNM header"};
        if (std::isspace(ch)) {
            ++c.i;
        } else if (ch == '#') {
            while (c.peek() != EOF && c.peek() != '\n') ++c.i;
        } else {
            break;
        }
    }
    if (!std::isdigit(c.peek()) && c.peek() != '+' && c.peek() != '-') throw IoFail{"malformed PNM header"};
    long v = 0;
    bool neg = false;
    if (c.peek() == '+' || c.peek() == '-') neg = c.b[c.i++] == '-';
    if (!std::isdigit(c.peek())) throw IoFail{"malformed PNM header"};
    while (std::isdigit(c.peek())) {
        v = v * 10 + (c.b[c.i++] - '0');
        if (v > (1L << 30)) throw IoFail{"malformed PNM header"};
    }
    return (int)(neg ? -v : v);
}

void load_pnm(const std::string& path, std::vector<float>& img, int& w, int& h) {
    const std::vector<uint8_t> b = read_file(path);
    Cursor c{b};
    if (b.size() < 2 || b[0] != 'P' || b[1] < '2' || b[1] > '6')
        throw IoFail{"unsupported PNM format in " + path};
    const char kind = (char)b[1];
    if (kind == '4') throw IoFail{"unsupported PNM format in " + path};
    c.i = 2;
    w = next_pnm_int(c);
    h = next_pnm_int(c);
    const int maxval = next_pnm_int(c);
    if (w < 1 || h < 1 || maxval < 1 || maxval > 255) throw IoFail{"unsupported PNM dimensions in " + path};
    const size_t n = (size_t)w * h;
    img.assign(n, 0.f);
    const int ch = (kind == '3' || kind == '6') ? 3 : 1;
    if (kind == '2' || kind == '3') {  // ASCII samples
        for (size_t i = 0; i < n; ++i) {
            int v[3];
            for (int k = 0; k < ch; ++k) {
                while (c.peek() != EOF && std::isspace(c.peek())) ++c.i;
                if (c.peek() == EOF) throw IoFail{"truncated PNM data in " + path};
                try {
                    v[k] = next_pnm_int(c);
                } catch (const IoFail&) {
                    throw IoFail{"truncated PNM data in " + path};
                }
            }
            img[i] = ch == 3 ? luminance(v[0], v[1], v[2]) : (float)v[0];
        }
    } else {  // binary: a single whitespace byte after maxval
        ++c.i;
        if (b.size() < c.i + n * ch) throw IoFail{"truncated PNM data in " + path};
        const uint8_t* raw = b.data() + c.i;
        for (size_t i = 0; i < n; ++i)
            img[i] = ch == 3 ? luminance(raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]) : (float)raw[i];
    }
}

void save_pgm(const float* img, int w, int h, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoFail{"cannot write image: " + path};
    out << "P5\n" << w << " " << h << "\n255\n";
    std::vector<uint8_t> raw((size_t)w * h);
    for (size_t i = 0; i < raw.size(); ++i) raw[i] = quantize(img[i]);
    out.write(reinterpret_cast<const char*>(raw.data()), (std::streamsize)raw.size());
    if (!out) throw IoFail{"cannot write image: " + path};
}

// ------------------------------------------------------------------ PNG

uint32_t be32(const uint8_t* p) { return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | p[3]; }

int paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

// Undo the scanline filters of one (sub)image in place: `data` holds h rows of
// 1 + rowbytes bytes; returns the unfiltered rows (h x rowbytes).
std::vector<uint8_t> unfilter(const uint8_t* data, size_t rowbytes, int h, int bpp) {
    std::vector<uint8_t> out(rowbytes * h);
    for (int y = 0; y < h; ++y) {
        const uint8_t ft = data[y * (rowbytes + 1)];
        const uint8_t* in = data + y * (rowbytes + 1) + 1;
        uint8_t* row = out.data() + y * rowbytes;
        const uint8_t* up = y ? row - rowbytes : nullptr;
        for (size_t x = 0; x < rowbytes; ++x) {
            const int a = x >= (size_t)bpp ? row[x - bpp] : 0, b = up ? up[x] : 0;
            const int c = (up && x >= (size_t)bpp) ? up[x - bpp] : 0;
            int v = in[x];
            switch (ft) {
                case 0: break;
                case 1: v += a; break;
                case 2: v += b; break;
                case 3: v += (a + b) >> 1; break;
                case 4: v += paeth(a, b, c); break;
                default: throw IoFail{"bad PNG filter"};
            }
            row[x] = (uint8_t)v;
        }
    }
    return out;
}

void load_png(const std::string& path, std::vector<float>& img, int& w, int& h) {
    const std::vector<uint8_t> b = read_file(path);
    static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    if (b.size() < 8 || std::memcmp(b.data(), sig, 8) != 0) throw IoFail{"failed to decode PNG: " + path};
    size_t i = 8;
    int depth = 0, ctype = -1, interlace = 0;
    w = h = 0;
    std::vector<uint8_t> idat, plte;
    while (i + 12 <= b.size()) {
        const uint32_t len = be32(&b[i]);
        if (i + 12 + (size_t)len > b.size()) throw IoFail{"failed to decode PNG: " + path};
        const char* type = reinterpret_cast<const char*>(&b[i + 4]);
        const uint8_t* d = &b[i + 8];
        if (!std::memcmp(type, "IHDR", 4) && len >= 13) {
            w = (int)be32(d);
            h = (int)be32(d + 4);
            depth = d[8];
            ctype = d[9];
            interlace = d[12];
        } else if (!std::memcmp(type, "PLTE", 4)) {
            plte.assign(d, d + len);
        } else if (!std::memcmp(type, "IDAT", 4)) {
            idat.insert(idat.end(), d, d + len);
        } else if (!std::memcmp(type, "IEND", 4)) {
            break;
        }
        i += 12 + len;
    }
    const bool ok_type = (ctype == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16)) ||
                         (ctype == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                         ((ctype == 2 || ctype == 4 || ctype == 6) && (depth == 8 || depth == 16));
    if (w <= 0 || h <= 0 || !ok_type || interlace > 1 || (ctype == 3 && plte.empty()))
        throw IoFail{"failed to decode PNG: " + path};
    const int spp = ctype == 2 ? 3 : ctype == 4 ? 2 : ctype == 6 ? 4 : 1;  // samples per pixel
    const int bits = spp * depth, bpp = std::max(1, bits / 8);
    // inflate
    z_stream zs;
    std::memset(&zs, 0, sizeof zs);
    if (inflateInit(&zs) != Z_OK) throw IoFail{"failed to decode PNG: " + path};
    // the exact size of the filtered data (all passes)
    static const int ax0[7] = {0, 4, 0, 2, 0, 1, 0}, ay0[7] = {0, 0, 4, 0, 2, 0, 1};
    static const int adx[7] = {8, 8, 4, 4, 2, 2, 1}, ady[7] = {8, 8, 8, 4, 4, 2, 2};
    struct Pass {
        int pw, ph;
        size_t rowbytes;
    };
    std::vector<Pass> passes;
    size_t total = 0;
    for (int p = 0; p < (interlace ? 7 : 1); ++p) {
        Pass ps;
        ps.pw = interlace ? (w - ax0[p] + adx[p] - 1) / adx[p] : w;
        ps.ph = interlace ? (h - ay0[p] + ady[p] - 1) / ady[p] : h;
        if (ps.pw <= 0 || ps.ph <= 0) ps.pw = ps.ph = 0;
        ps.rowbytes = ((size_t)ps.pw * bits + 7) / 8;
        if (ps.pw) total += (ps.rowbytes + 1) * ps.ph;
        passes.push_back(ps);
    }
    std::vector<uint8_t> raw(total);
    zs.next_in = idat.data();
    zs.avail_in = (uInt)idat.size();
    zs.next_out = raw.data();
    zs.avail_out = (uInt)raw.size();
    const int zr = inflate(&zs, Z_FINISH);
    const bool full = zs.avail_out == 0;
    inflateEnd(&zs);
    if (!full || (zr != Z_STREAM_END && zr != Z_OK && zr != Z_BUF_ERROR)) throw IoFail{"failed to decode PNG: " + path};
    // 8-bit samples per pixel after the reference's transforms
    std::vector<uint8_t> px((size_t)w * h * 3);
    int chans = 0;  // 1 = gray, 3 = rgb after the transforms
    auto sample = [&](const uint8_t* row, int x, int s) -> int {
        if (depth == 16) return row[(x * spp + s) * 2];  // png_set_strip_16: high byte
        if (depth == 8) return row[x * spp + s];
        const int per = 8 / depth, shift = 8 - depth * (x % per + 1);
        return (row[x / per] >> shift) & ((1 << depth) - 1);
    };
    size_t off = 0;
    for (int p = 0; p < (int)passes.size(); ++p) {
        const Pass& ps = passes[p];
        if (!ps.pw) continue;
        const std::vector<uint8_t> rows = unfilter(raw.data() + off, ps.rowbytes, ps.ph, bpp);
        off += (ps.rowbytes + 1) * ps.ph;
        for (int yy = 0; yy < ps.ph; ++yy) {
            const uint8_t* row = rows.data() + yy * ps.rowbytes;
            const int y = interlace ? ay0[p] + yy * ady[p] : yy;
            for (int xx = 0; xx < ps.pw; ++xx) {
                const int x = interlace ? ax0[p] + xx * adx[p] : xx;
                uint8_t* o = &px[((size_t)y * w + x) * 3];
                if (ctype == 3) {  // palette -> RGB (png_set_palette_to_rgb)
                    const int k = sample(row, xx, 0);
                    if ((size_t)(3 * k + 2) >= plte.size()) throw IoFail{"failed to decode PNG: " + path};
                    o[0] = plte[3 * k];
                    o[1] = plte[3 * k + 1];
                    o[2] = plte[3 * k + 2];
                    chans = 3;
                } else if (ctype == 2 || ctype == 6) {
                    o[0] = (uint8_t)sample(row, xx, 0);
                    o[1] = (uint8_t)sample(row, xx, 1);
                    o[2] = (uint8_t)sample(row, xx, 2);
                    chans = 3;
                } else {  // gray (+alpha): 1/2/4-bit gray scaled to 8 bits (png_set_expand_gray_1_2_4_to_8)
                    int v = sample(row, xx, 0);
                    if (depth < 8) v = v * 255 / ((1 << depth) - 1);
                    o[0] = (uint8_t)v;
                    chans = 1;
                }
            }
        }
    }
    img.assign((size_t)w * h, 0.f);
    for (size_t k = 0; k < img.size(); ++k) {
        const uint8_t* o = &px[k * 3];
        img[k] = chans == 3 ? luminance(o[0], o[1], o[2]) : (float)o[0];
    }
}

void put32(std::vector<uint8_t>& v, uint32_t x) {
    v.push_back((uint8_t)(x >> 24));
    v.push_back((uint8_t)(x >> 16));
    v.push_back((uint8_t)(x >> 8));
    v.push_back((uint8_t)x);
}

void chunk(std::vector<uint8_t>& out, const char* type, const std::vector<uint8_t>& data) {
    put32(out, (uint32_t)data.size());
    const size_t t0 = out.size();
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), data.begin(), data.end());
    put32(out, (uint32_t)crc32(0, out.data() + t0, (uInt)(out.size() - t0)));
}

void save_png(const uint8_t* px, int w, int h, int chans, const std::string& path) {
    std::vector<uint8_t> filt;
    filt.reserve(((size_t)w * chans + 1) * h);
    for (int y = 0; y < h; ++y) {
        filt.push_back(0);
        filt.insert(filt.end(), px + (size_t)y * w * chans, px + (size_t)(y + 1) * w * chans);
    }
    uLongf zn = compressBound((uLong)filt.size());
    std::vector<uint8_t> z(zn);
    if (compress2(z.data(), &zn, filt.data(), (uLong)filt.size(), Z_DEFAULT_COMPRESSION) != Z_OK)
        throw IoFail{"failed to encode PNG: " + path};
    z.resize(zn);
    std::vector<uint8_t> out = {137, 80, 78, 71, 13, 10, 26, 10};
    std::vector<uint8_t> ihdr;
    put32(ihdr, (uint32_t)w);
    put32(ihdr, (uint32_t)h);
    ihdr.insert(ihdr.end(), {8, (uint8_t)(chans == 3 ? 2 : 0), 0, 0, 0});
    chunk(out, "IHDR", ihdr);
    chunk(out, "IDAT", z);
    chunk(out, "IEND", {});
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoFail{"cannot write image: " + path};
    f.write(reinterpret_cast<const char*>(out.data()), (std::streamsize)out.size());
    if (!f) throw IoFail{"cannot write image: " + path};
}

}  // namespace

extern "C" {

int xa_load_image(const char* path, float* out, size_t cap, int* w, int* h) {
    *w = *h = 0;
    try {
        const std::string p(path ? path : "");
        std::vector<float> img;
        int iw = 0, ih = 0;
        if (has_suffix(p, ".png"))
            load_png(p, img, iw, ih);
        else if (has_suffix(p, ".pgm") || has_suffix(p, ".ppm") || has_suffix(p, ".pnm"))
            load_pnm(p, img, iw, ih);
        else
            throw IoFail{"unsupported image format: " + p};
        *w = iw;
        *h = ih;
        if (!out) return XA_OK;
        if (cap < img.size()) return xa::host_error(XA_ECAPACITY, "load_image: output capacity");
        std::memcpy(out, img.data(), img.size() * sizeof(float));
        return XA_OK;
    } catch (const IoFail& e) {
        return xa::host_error(XA_EIO, e.msg);
    } catch (const std::exception& e) {
        return xa::host_error(XA_EIO, e.what());
    }
}

int xa_save_image(const float* img, int w, int h, const char* path) {
    try {
        const std::string p(path ? path : "");
        if (!img || w <= 0 || h <= 0) return xa::host_error(XA_EINVAL, "save_image: empty image");
        if (has_suffix(p, ".png")) {
            std::vector<uint8_t> q((size_t)w * h);
            for (size_t i = 0; i < q.size(); ++i) q[i] = quantize(img[i]);
            save_png(q.data(), w, h, 1, p);
        } else if (has_suffix(p, ".pgm")) {
            save_pgm(img, w, h, p);
        } else {
            throw IoFail{"unsupported output format: " + p};
        }
        return XA_OK;
    } catch (const IoFail& e) {
        return xa::host_error(XA_EIO, e.msg);
    }
}

int xa_save_png_rgb(const uint8_t* rgb, int w, int h, const char* path) {
    try {
        if (!rgb || w <= 0 || h <= 0) return xa::host_error(XA_EINVAL, "save_png_rgb: empty image");
        save_png(rgb, w, h, 3, std::string(path ? path : ""));
        return XA_OK;
    } catch (const IoFail& e) {
        return xa::host_error(XA_EIO, e.msg);
    }
}

int xa_quantize(const float* img, size_t n, uint8_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = quantize(img[i]);
    return XA_OK;
}

}  // extern "C"
