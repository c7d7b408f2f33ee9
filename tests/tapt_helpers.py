"""Shared helpers for the parity tests: build the same problem for the device engine and
for the oracle restatement, and run the oracle's PT schedule."""
import numpy as np

from oracle import oracle as O


def geometric(b0, b1, R):
    return b0 * (b1 / b0) ** (np.arange(R) / (R - 1.0))


def linear(b0, b1, R):
    return np.linspace(b0, b1, R)


def oracle_lattice(dims):
    return O.lattice_graph(dims)


def oracle_ea(dims, disorder_seed, gid):
    return O.ea_graph(dims, disorder_seed, gid)


def run_oracle(graphs, betas, seed, gid0, order_fn, n_sweeps, swap_every=1, measure_every=0, measure_from=0,
               props=None, e_lo=0, width=1, nbins=0):
    """Run the restated PT schedule for each instance graph; returns the PT objects.
    props: dict(every=k, targets=n_targets, m_bias=array, refine=int) for synthetic TAPT rounds."""
    pts = []
    for k, g in enumerate(graphs):
        pt = O.PT(g, betas, seed, gid0 + k, order_fn(g))
        if props:
            pt.run(n_sweeps, swap_every, props["every"], props["targets"], props.get("m_bias"), props["refine"],
                   measure_every, measure_from, e_lo, width, nbins)
        else:
            pt.run(n_sweeps, swap_every, 0, 0, None, 0, measure_every, measure_from, e_lo, width, nbins)
        pts.append(pt)
    return pts


def colour_order_for(model_colours):
    def f(g):
        return g.colour_order(model_colours)
    return f


def checkerboard_order(dims):
    cols = O.checkerboard_colours(dims)

    def f(g):
        return g.colour_order(cols)
    return f


def index_order(g):
    return g.index_order()
