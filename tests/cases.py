"""Case builders for tests (inputs only; no method arithmetic)."""
import numpy as np

import gen


def small_random_mesh(nx=5, ny=5, nz=2, jitter=0.3, seed=11, permute=True):
    """A perturbed, randomly permuted hex mesh (<= ~50 cells) for brute-force pins."""
    m = gen.box(nx, ny, nz, (1.0, 1.0, 0.5), jitter=jitter, seed=seed)
    if permute:
        m = gen.permute(m, seed=seed + 100)
    return m


def dirichlet_box(nx, ny, nz, L=(1.0, 1.0, 1.0), walls=("xmin", "xmax", "ymin", "ymax", "zmin", "zmax"), empty=()):
    m = gen.box(nx, ny, nz, L)
    for p in m.patches:
        if p.name in empty:
            m = gen.set_kind(m, p.name, gen.EMPTY)
        elif p.name in walls:
            m = gen.set_kind(m, p.name, gen.FIXED_VALUE, np.zeros(p.n_faces))
    return m


def dense_ldu(n, owner, neighbour, diag, upper, lower=None):
    """Dense matrix straight from the lduMatrix definition: numpy, independent of oracle.c."""
    lower = upper if lower is None else lower
    A = np.zeros((n, n))
    A[np.arange(n), np.arange(n)] = diag
    np.add.at(A, (np.asarray(owner), np.asarray(neighbour)), upper)
    np.add.at(A, (np.asarray(neighbour), np.asarray(owner)), lower)
    return A


def lattice_modes(dims, ks, kind):
    """Separable sin (Dirichlet) / cos (Neumann) modes on a lattice, cell id i + nx(j + ny k)."""
    u = np.ones(1)
    for n, k in zip(dims, ks):  # x fastest -> build with kron in reverse
        i = np.arange(n)
        f = np.sin(np.pi * k * (i + 0.5) / n) if kind == "sin" else np.cos(np.pi * k * (i + 0.5) / n)
        u = np.kron(f, u)
    return u


def eigenvalue(dims, ks, coefs):
    """lambda = -sum_d coef_d 4 sin^2(pi k_d / (2 n_d)) (ghost-mirror identity)."""
    return -sum(c * 4.0 * np.sin(np.pi * k / (2.0 * n)) ** 2 for n, k, c in zip(dims, ks, coefs))


def asym_system(mesh, seed=0, skew=0.4):
    """Test input for the asymmetric solvers (§8(f3)): the Laplacian's coefficients made
    asymmetric like a convection-diffusion operator, upper = u (1 + e), lower = u (1 - e),
    e ~ U(-skew, skew) per face, and a diagonal that dominates the row sums by 5 %
    (negative, like the Laplacian).  Returns (diag, upper, lower, source)."""
    import oracle as O
    s = O.assemble(mesh, None, -1)
    rng = np.random.default_rng(seed)
    e = rng.uniform(-skew, skew, mesh.n_faces)
    upper, lower = s.upper * (1 + e), s.upper * (1 - e)
    off = np.zeros(mesh.n_cells)
    np.add.at(off, mesh.owner, np.abs(upper))
    np.add.at(off, mesh.neighbour, np.abs(lower))
    diag = -1.05 * np.maximum(off, 1e-12)
    return diag, upper, lower, rng.standard_normal(mesh.n_cells) * mesh.V


def asym_decomposed(mesh, part, seed=0, skew=0.4, sym=False):
    """The asym_system of `mesh` split over the parts of `part` (gen.decompose): per domain
    dict(diag, upper, lower, source, iface, iface_t) -- processor faces carry A[P][N] = upper
    and A[N][P] = lower of the undecomposed face, oriented by is_owner (Amul: own row's entry,
    Tmul: the remote row's entry).  sym: lower = upper.  Returns (subs, systems, global)."""
    import gen
    d, u, l, b = asym_system(mesh, seed=seed, skew=skew)
    if sym:
        l = u.copy()
    P = int(part.max()) + 1
    subs = gen.decompose(mesh, part, P)
    gidx = {int(f): i for i, f in enumerate(mesh.gface)}
    loc = {int(g): i for i, g in enumerate(mesh.gid)}
    systems = []
    for sm in subs:
        fi = np.array([gidx[int(f)] for f in sm.gface], dtype=np.int64)
        assert np.array_equal(mesh.gid[mesh.owner[fi]], sm.gid[sm.owner])  # orientation kept
        ci = np.array([loc[int(g)] for g in sm.gid], dtype=np.int64)
        iface, iface_t = [], []
        for pt in sm.patches:
            if pt.kind != gen.PROCESSOR:
                continue
            gi = np.array([gidx[int(f)] for f in pt.global_face], dtype=np.int64)
            own = np.asarray(pt.is_owner, bool)
            iface.append(np.where(own, u[gi], l[gi]))
            iface_t.append(np.where(own, l[gi], u[gi]))
        systems.append(dict(diag=d[ci], upper=u[fi], lower=l[fi], source=b[ci], iface=iface, iface_t=iface_t))
    return subs, systems, (d, u, l, b)
