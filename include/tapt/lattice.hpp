// tapt/lattice.hpp -- drop-in for LatticeSpec (proj/include/tapt/lattice.hpp:15-39,
// proj/src/lattice.cpp).  Site order: grid2d raster row-major (index = row*lx + col),
// grid3d x-fastest (index = x + L*(y + L*z)); periodic wrap bonds only when the extent is > 2.
// Graphs built here carry a lattice tag, so periodic power-of-two lattices run on the
// bit-sliced stencil kernel (K1) instead of the general CSR kernel.
#pragma once

#include <map>

#include "tapt/spin_model.hpp"

namespace tapt {

struct LatticeSpec {
    enum class Kind { grid2d, grid3d };
    enum class Boundary { open, periodic };

    Kind kind = Kind::grid2d;
    Boundary boundary = Boundary::open;
    int ly = 0, lx = 0;
    int l = 0;
    double coupling = 1.0;

    static LatticeSpec grid2d(int ly, int lx, double j = 1.0, Boundary b = Boundary::open) {
        if (ly < 1 || lx < 1) throw ConfigError("grid2d dimensions must be >= 1");
        LatticeSpec s;
        s.kind = Kind::grid2d;
        s.boundary = b;
        s.ly = ly;
        s.lx = lx;
        s.coupling = j;
        return s;
    }
    static LatticeSpec grid3d(int l, double j = 1.0, Boundary b = Boundary::open) {
        if (l < 1) throw ConfigError("grid3d size must be >= 1");
        LatticeSpec s;
        s.kind = Kind::grid3d;
        s.boundary = b;
        s.l = l;
        s.coupling = j;
        return s;
    }

    std::size_t n_sites() const {
        return kind == Kind::grid2d ? static_cast<std::size_t>(ly) * lx : static_cast<std::size_t>(l) * l * l;
    }
    // Bond count as graph() builds it (wrap bonds need extent > 2).
    std::size_t n_edges() const {
        const bool per = boundary == Boundary::periodic;
        auto along = [per](std::size_t extent, std::size_t lines) {
            std::size_t e = lines * (extent - 1);
            if (per && extent > 2) e += lines;
            return e;
        };
        if (kind == Kind::grid2d)
            return along(lx, ly) + along(ly, lx);
        const std::size_t p = static_cast<std::size_t>(l) * l;
        return 3 * along(l, p);
    }
    std::uint32_t index2d(int row, int col) const { return static_cast<std::uint32_t>(row * lx + col); }
    std::uint32_t index3d(int x, int y, int z) const {
        return static_cast<std::uint32_t>(x + l * (y + static_cast<long>(l) * z));
    }

    CouplingGraph graph() const { return graph_clamped({}); }

    CouplingGraph graph_clamped(const std::map<std::uint32_t, int>& clamp) const {
        CouplingGraph::Builder b(n_sites());
        const bool per = boundary == Boundary::periodic;
        auto link = [&](std::uint32_t i, int coord, int extent, std::uint32_t next, std::uint32_t first) {
            if (coord + 1 < extent)
                b.add_coupling(i, next, coupling);
            else if (per && extent > 2)
                b.add_coupling(i, first, coupling);
        };
        if (kind == Kind::grid2d) {
            for (int r = 0; r < ly; ++r)
                for (int c = 0; c < lx; ++c) {
                    const std::uint32_t i = index2d(r, c);
                    link(i, c, lx, c + 1 < lx ? index2d(r, c + 1) : 0, index2d(r, 0));
                    link(i, r, ly, r + 1 < ly ? index2d(r + 1, c) : 0, index2d(0, c));
                }
        } else {
            for (int z = 0; z < l; ++z)
                for (int y = 0; y < l; ++y)
                    for (int x = 0; x < l; ++x) {
                        const std::uint32_t i = index3d(x, y, z);
                        link(i, x, l, x + 1 < l ? index3d(x + 1, y, z) : 0, index3d(0, y, z));
                        link(i, y, l, y + 1 < l ? index3d(x, y + 1, z) : 0, index3d(x, 0, z));
                        link(i, z, l, z + 1 < l ? index3d(x, y, z + 1) : 0, index3d(x, y, 0));
                    }
        }
        for (const auto& [site, v] : clamp) b.set_clamp(site, v);
        CouplingGraph g = b.build();
        if (kind == Kind::grid2d)
            g.tag_lattice({2, ly, lx, 1, coupling, per});
        else
            g.tag_lattice({3, l, l, l, coupling, per});
        return g;
    }
};

template <typename PatternFn>
std::map<std::uint32_t, int> top_rows_clamp(const LatticeSpec& spec, int rows, PatternFn pattern) {
    std::map<std::uint32_t, int> clamp;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < spec.lx; ++c) clamp[spec.index2d(r, c)] = pattern(r, c);
    return clamp;
}

}  // namespace tapt
