// Host services behind the C ABI that are not on the device hot path:
// seeded instances (bit-exact with ref instance.cpp so GPU inputs equal
// oracle inputs), generator validation, JSON fixtures, the dense O(s^2)
// reference multiply and the closed-form cost model. These are setup /
// oracle-side ABI functions (SURVEY.md §2 "ABI-required"); the split matvec
// itself never runs here.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numbers>
#include <sstream>
#include <thread>

#include "host.hpp"

namespace tsb {

int64_t volume(const Shape& s)
{
    int64_t v = 1;
    for (auto n : s)
        v *= n;
    return v;
}

Shape check_levels(int32_t d, const int64_t* levels)
{
    if (d < 1 || !levels)
        fail(TS_ERR_INVALID_ARGUMENT, "levels must hold d >= 1 sizes");
    if (d > 31)
        fail(TS_ERR_SHAPE, "at most 31 levels are supported (branch ids are 32-bit)");
    Shape s(levels, levels + d);
    for (auto n : s)
        if (n < 1)
            fail(TS_ERR_SHAPE, "level sizes must be >= 1");
    return s;
}

std::vector<int> signs_for_mode(int d, ts_symmetry mode)
{
    const int s = mode == TS_SYM_SYMMETRIC ? 1 : (mode == TS_SYM_SKEW ? -1 : 0);
    return std::vector<int>(static_cast<size_t>(d), s);
}

// ref generator.cpp:38-62 with a per-axis sign: exact comparison of each lag
// with its single-axis mirror.
void validate_symmetry(const Shape& levels, const std::vector<cplx>& lags,
                       const std::vector<int>& axis_sign)
{
    const int d = static_cast<int>(levels.size());
    Shape ls(levels.size());
    for (int a = 0; a < d; ++a)
        ls[a] = 2 * levels[a] - 1;
    for (int a = 0; a < d; ++a) {
        if (axis_sign[a] == 0)
            continue;
        int64_t inner = 1, outer = 1;
        for (int b = a + 1; b < d; ++b)
            inner *= ls[b];
        for (int b = 0; b < a; ++b)
            outer *= ls[b];
        const int64_t len = ls[a];
        for (int64_t o = 0; o < outer; ++o)
            for (int64_t k = 0; k < len; ++k)
                for (int64_t i = 0; i < inner; ++i) {
                    const cplx& l = lags[(o * len + k) * inner + i];
                    const cplx& r = lags[(o * len + (len - 1 - k)) * inner + i];
                    if (axis_sign[a] > 0 ? (l != r) : (l != -r))
                        fail(TS_ERR_SYMMETRY,
                             axis_sign[a] > 0
                                 ? "symmetric mode requires t_m == t_{-m} per level"
                                 : "skew mode requires t_m == -t_{-m} per level (t_0 == 0)");
                }
    }
}

Generator make_generator(Shape levels, std::vector<cplx> lags, ts_symmetry sym)
{
    if (sym != TS_SYM_GENERAL && sym != TS_SYM_SYMMETRIC && sym != TS_SYM_SKEW)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid symmetry value");
    int64_t expect = 1;
    for (auto n : levels)
        expect *= 2 * n - 1;
    if (static_cast<int64_t>(lags.size()) != expect)
        fail(TS_ERR_SHAPE, "lag tensor must have shape (2n-1) per level");
    validate_symmetry(levels, lags, signs_for_mode(static_cast<int>(levels.size()), sym));
    Generator g;
    g.levels = std::move(levels);
    g.lags = std::move(lags);
    g.symmetry = sym;
    return g;
}

BlockGenerator block_from_scalar(const Generator& g)
{
    BlockGenerator b;
    b.levels = g.levels;
    b.m = 1;
    b.n_unique = 1;
    b.comp_map = {0};
    b.lags = {g.lags};
    b.axis_sign = signs_for_mode(static_cast<int>(g.levels.size()), g.symmetry);
    b.scalar_symmetry = g.symmetry;
    return b;
}

BlockGenerator block_dyadic(const Shape& levels, double k, cplx self_term)
{
    const int d = static_cast<int>(levels.size());
    if (d != 3)
        fail(TS_ERR_SHAPE, "the dyadic Green kernel is defined for d = 3");
    if (!(k > 0.0) || !std::isfinite(k))
        fail(TS_ERR_INVALID_ARGUMENT, "dyadic wavenumber must be positive");
    BlockGenerator b;
    b.levels = levels;
    b.m = 3;
    b.n_unique = 6;
    b.dyadic = true;
    b.k = k;
    b.self_term = self_term;
    int u = 0;
    int map[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = i; j < 3; ++j) {
            map[i][j] = map[j][i] = u++;
            b.dyadic_ij.emplace_back(i, j);
        }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            b.comp_map.push_back(map[i][j]);
    // G_ij(m) is even along axis a unless exactly one of i, j equals a
    for (auto [i, j] : b.dyadic_ij)
        for (int a = 0; a < 3; ++a)
            b.axis_sign.push_back(((i == a) + (j == a)) % 2 ? -1 : 1);
    return b;
}

// ---- instances (ref instance.hpp:16-25, instance.cpp) ------------------

uint64_t SplitMix64::next()
{
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

SplitMix64 seeded_stream(uint64_t seed, uint64_t role)
{
    return SplitMix64(seed ^ ((role + 1) * 0x9E3779B97F4A7C15ull));
}

namespace {

class Gaussian {
  public:
    Gaussian(SplitMix64 rng, double variance) : rng_(rng)
    {
        if (!(variance >= 0.0))
            fail(TS_ERR_INVALID_ARGUMENT, "variance must be >= 0");
        sigma_ = std::sqrt(variance);
    }
    double next()
    {
        if (have_) {
            have_ = false;
            return spare_;
        }
        const double u1 = 1.0 - rng_.next_unit();
        const double u2 = rng_.next_unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * std::numbers::pi * u2;
        spare_ = sigma_ * r * std::sin(a);
        have_ = true;
        return sigma_ * r * std::cos(a);
    }

  private:
    SplitMix64 rng_;
    double sigma_ = 0.0, spare_ = 0.0;
    bool have_ = false;
};

// Orbit average over single-level lag negations (ref instance.cpp:43-103):
// each orbit is evaluated once at its canonical member (all lags >= 0) and
// written to every member with the exact sign character.
void symmetrize(std::vector<cplx>& lags, const Shape& levels, bool skew)
{
    const int d = static_cast<int>(levels.size());
    const uint32_t patterns = 1u << d;
    const double weight = 1.0 / static_cast<double>(patterns);
    Shape ls(levels.size());
    for (int a = 0; a < d; ++a)
        ls[a] = 2 * levels[a] - 1;
    std::vector<int64_t> idx(static_cast<size_t>(d), 0);
    auto member = [&](uint32_t sig, double& chi) {
        int64_t off = 0;
        chi = 1.0;
        for (int a = 0; a < d; ++a) {
            int64_t k = idx[a];
            if ((sig >> a) & 1u) {
                k = ls[a] - 1 - k;
                if (skew)
                    chi = -chi;
            }
            off = off * ls[a] + k;
        }
        return off;
    };
    const int64_t total = volume(ls);
    for (int64_t off = 0; off < total; ++off) {
        bool canonical = true, zero_lag = false;
        for (int a = 0; a < d; ++a) {
            canonical = canonical && idx[a] >= levels[a] - 1;
            zero_lag = zero_lag || idx[a] == levels[a] - 1;
        }
        if (canonical) {
            cplx acc{0.0, 0.0};
            double chi;
            if (!(skew && zero_lag))
                for (uint32_t sig = 0; sig < patterns; ++sig) {
                    const int64_t src = member(sig, chi);
                    acc += chi * weight * lags[src];
                }
            for (uint32_t sig = 0; sig < patterns; ++sig) {
                const int64_t dst = member(sig, chi);
                lags[dst] = chi * acc;
            }
        }
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < ls[a])
                break;
            idx[a] = 0;
        }
    }
}

}  // namespace

// Complex draws of one stream: element i consumes uniforms 2i and 2i+1 of
// the SplitMix64 sequence and is exactly one Box-Muller pair (cos part =
// real, cached sin part = imaginary), so the sequence splits into
// independent chunks via SplitMix64's additive state (jump = i * gamma).
// Bit-identical to the sequential GaussianStream of ref instance.cpp.
static void fill_complex_gaussian(cplx* out, int64_t count, uint64_t seed, uint64_t role,
                                  double variance)
{
    const uint64_t gamma = 0x9E3779B97F4A7C15ull;
    const uint64_t state0 = seeded_stream(seed, role).state;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nthreads = count < (int64_t(1) << 16) ? 1 : std::min<int64_t>(hw, 64);
    auto work = [&](int64_t b, int64_t e) {
        SplitMix64 rng(state0 + static_cast<uint64_t>(2 * b) * gamma);
        Gaussian gauss(rng, variance);
        for (int64_t i = b; i < e; ++i) {
            const double re = gauss.next();
            out[i] = cplx{re, gauss.next()};
        }
    };
    if (nthreads == 1) {
        work(0, count);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (count + nthreads - 1) / nthreads;
    for (int64_t t = 0; t < nthreads; ++t) {
        const int64_t b = t * chunk, e = std::min(count, b + chunk);
        if (b < e)
            th.emplace_back(work, b, e);
    }
    for (auto& t : th)
        t.join();
}

Generator random_generator(const Shape& levels, uint64_t seed, double variance, ts_symmetry sym)
{
    int64_t count = 1;
    for (auto n : levels)
        count *= 2 * n - 1;
    if (!(variance >= 0.0))
        fail(TS_ERR_INVALID_ARGUMENT, "variance must be >= 0");
    std::vector<cplx> lags(static_cast<size_t>(count));
    fill_complex_gaussian(lags.data(), count, seed, 0, variance);
    if (sym != TS_SYM_GENERAL)
        symmetrize(lags, levels, sym == TS_SYM_SKEW);
    return make_generator(levels, std::move(lags), sym);
}

std::vector<cplx> random_vector(const Shape& levels, uint64_t seed, double variance)
{
    if (!(variance >= 0.0))
        fail(TS_ERR_INVALID_ARGUMENT, "variance must be >= 0");
    std::vector<cplx> v(static_cast<size_t>(volume(levels)));
    fill_complex_gaussian(v.data(), static_cast<int64_t>(v.size()), seed, 1, variance);
    return v;
}

void random_vector_into(const Shape& levels, uint64_t seed, double variance, cplx* out)
{
    if (!(variance >= 0.0))
        fail(TS_ERR_INVALID_ARGUMENT, "variance must be >= 0");
    fill_complex_gaussian(out, volume(levels), seed, 1, variance);
}

// ---- JSON fixtures (format of ref proj/README.md:144-156) --------------

namespace {

struct JsonCursor {
    const std::string& s;
    size_t i = 0;
    void ws()
    {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r'))
            ++i;
    }
    [[noreturn]] void bad(const char* what) const
    {
        fail(TS_ERR_IO, std::string("generator json parse error: ") + what + " at offset " +
                            std::to_string(i));
    }
    void expect(char c)
    {
        ws();
        if (i >= s.size() || s[i] != c)
            bad("unexpected character");
        ++i;
    }
    bool peek(char c)
    {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string str()
    {
        expect('"');
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\' && i + 1 < s.size())
                ++i;
            out += s[i++];
        }
        if (i >= s.size())
            bad("unterminated string");
        ++i;
        return out;
    }
    double num()
    {
        ws();
        const char* b = s.c_str() + i;
        char* e = nullptr;
        const double v = std::strtod(b, &e);
        if (e == b)
            bad("expected a number");
        i += static_cast<size_t>(e - b);
        return v;
    }
    void skip_value()
    {
        ws();
        if (peek('{')) {
            expect('{');
            if (peek('}')) {
                ++i;
                return;
            }
            do {
                str();
                expect(':');
                skip_value();
            } while (peek(',') && (++i, true));
            expect('}');
        } else if (peek('[')) {
            expect('[');
            if (peek(']')) {
                ++i;
                return;
            }
            do
                skip_value();
            while (peek(',') && (++i, true));
            expect(']');
        } else if (peek('"')) {
            str();
        } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 4, "null") == 0) {
            i += 4;
        } else if (s.compare(i, 5, "false") == 0) {
            i += 5;
        } else {
            num();
        }
    }
};

}  // namespace

Generator generator_from_json(const std::string& text)
{
    JsonCursor c{text};
    Shape levels;
    std::vector<cplx> lags;
    std::string sym;
    bool have_l = false, have_g = false, have_s = false;
    c.expect('{');
    if (!c.peek('}')) {
        do {
            const std::string key = c.str();
            c.expect(':');
            if (key == "levels") {
                have_l = true;
                c.expect('[');
                if (!c.peek(']'))
                    do
                        levels.push_back(static_cast<int64_t>(c.num()));
                    while (c.peek(',') && (++c.i, true));
                c.expect(']');
            } else if (key == "lags") {
                have_g = true;
                c.expect('[');
                if (!c.peek(']'))
                    do {
                        if (!c.peek('['))
                            fail(TS_ERR_IO, "generator json lag entries must be [re, im] pairs");
                        c.expect('[');
                        const double re = c.num();
                        c.expect(',');
                        const double im = c.num();
                        if (!c.peek(']'))
                            fail(TS_ERR_IO, "generator json lag entries must be [re, im] pairs");
                        c.expect(']');
                        lags.emplace_back(re, im);
                    } while (c.peek(',') && (++c.i, true));
                c.expect(']');
            } else if (key == "symmetry") {
                have_s = true;
                sym = c.str();
            } else {
                c.skip_value();
            }
        } while (c.peek(',') && (++c.i, true));
    }
    c.expect('}');
    if (!have_l || !have_g || !have_s)
        fail(TS_ERR_IO, "generator json must contain levels, lags, symmetry");
    ts_symmetry mode;
    if (sym == "general")
        mode = TS_SYM_GENERAL;
    else if (sym == "symmetric")
        mode = TS_SYM_SYMMETRIC;
    else if (sym == "skew")
        mode = TS_SYM_SKEW;
    else
        fail(TS_ERR_INVALID_ARGUMENT, "unknown symmetry mode: " + sym);
    check_levels(static_cast<int32_t>(levels.size()), levels.data());
    return make_generator(std::move(levels), std::move(lags), mode);
}

std::string generator_to_json(const Generator& g)
{
    std::ostringstream os;
    char buf[64];
    os << "{\"lags\":[";
    for (size_t i = 0; i < g.lags.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%s[%.17g,%.17g]", i ? "," : "", g.lags[i].real(),
                      g.lags[i].imag());
        os << buf;
    }
    os << "],\"levels\":[";
    for (size_t a = 0; a < g.levels.size(); ++a)
        os << (a ? "," : "") << g.levels[a];
    os << "],\"symmetry\":\""
       << (g.symmetry == TS_SYM_SYMMETRIC ? "symmetric"
                                          : (g.symmetry == TS_SYM_SKEW ? "skew" : "general"))
       << "\"}";
    return os.str();
}

// ---- dense reference multiply (ref engine_embed.cpp:190-227) ------------

std::vector<cplx> naive_matvec(const Generator& g, const cplx* v, int64_t cap)
{
    const int64_t s = volume(g.levels);
    if (s > cap)
        fail(TS_ERR_CAP_EXCEEDED, "dense oracle cap exceeded: s = " + std::to_string(s) +
                                      " > cap = " + std::to_string(cap));
    const int d = static_cast<int>(g.levels.size());
    std::vector<cplx> y(static_cast<size_t>(s));
    std::vector<int64_t> jdx(static_cast<size_t>(d), 0), kdx(static_cast<size_t>(d), 0);
    for (int64_t j = 0; j < s; ++j) {
        cplx acc{0.0, 0.0};
        std::fill(kdx.begin(), kdx.end(), 0);
        for (int64_t k = 0; k < s; ++k) {
            int64_t off = 0;
            for (int a = 0; a < d; ++a) {
                const int64_t n = g.levels[a];
                off = off * (2 * n - 1) + (jdx[a] - kdx[a] + n - 1);
            }
            acc += g.lags[off] * v[k];
            for (int a = d - 1; a >= 0; --a) {
                if (++kdx[a] < g.levels[a])
                    break;
                kdx[a] = 0;
            }
        }
        y[j] = acc;
        for (int a = d - 1; a >= 0; --a) {
            if (++jdx[a] < g.levels[a])
                break;
            jdx[a] = 0;
        }
    }
    return y;
}

// ---- closed-form model (ref analysis.cpp:21-56) ------------------------

ts_complexity predict(int32_t d, double n)
{
    if (d < 1)
        fail(TS_ERR_INVALID_ARGUMENT, "complexity model requires d >= 1");
    if (!(n >= 2.0))
        fail(TS_ERR_INVALID_ARGUMENT, "ratio model requires n >= 2");
    ts_complexity r{};
    const double s = std::pow(n, d), p = std::pow(2.0, d);
    r.d = d;
    r.n = n;
    r.s = s;
    r.c_embed = 2.0 * p * s * std::log2(p * s) + p * s;
    r.c_split = 2.0 * (p - 1.0) * s * (2.0 * std::log2(n) + 1.0) + p * s;
    r.r_c = (d * std::log2(2.0 * n) + 1.0) / ((1.0 - 1.0 / p) * (2.0 * std::log2(n) + 1.0) + 1.0);
    r.r_c_asymptote = d / (2.0 - std::pow(2.0, -d + 1));
    r.r_m = 2.0 / ((d + 1.0) / p + 1.0);
    r.r_m_sym = (p + 1.0) / (d + 2.0);
    return r;
}

}  // namespace tsb
