"""Mutation sanity check for the oracle pins: each plausible mistake (dropped term, wrong sign,
wrong index, transposed operand) injected into oracle.c must fail at least one -m "not gpu" test.
Restores oracle.c at the end.  Run: python tests/tools/oracle_mutation_check.py"""
import subprocess, sys
import os
os.chdir(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
src = open('oracle/oracle.c').read()
muts = [
 ("diag[neighbour[f]] -= upper[f];", "/*dropped*/"),
 ("source[P] += (-gms) * (bdelta[i] * bvalue[i]);", "source[P] += (gms) * (bdelta[i] * bvalue[i]);"),
 ("diag[ref_cell] += diag[ref_cell];", ";"),
 ("*weight = den > 1e-150 ? SfdNei / den : 0.5;", "*weight = den > 1e-150 ? SfdOwn / den : 0.5;"),
 ("double beta = wArA / wArAold;", "double beta = wArAold / wArA;"),
 ("W[p].rA[c] -= alpha * W[p].wA[c];", "W[p].rA[c] += alpha * W[p].wA[c];"),
 ("s += fabs(W[p].wA[c] - xref) + fabs(D[p].source[c] - xref);", "s += fabs(W[p].wA[c] - xref);"),
 ("y[iface_cells[i]] += iface_coeffs[i] * x_remote[i];", "y[iface_cells[i]] += iface_coeffs[i] * x[iface_cells[i]];"),
 ("perm[queue[i]] = n_cells - 1 - i;", "perm[queue[i]] = i;"),
 ("return x->face < y->face ? -1 : (x->face > y->face);", "return x->face > y->face ? -1 : (x->face < y->face);"),
 ("for (int k = 0; k < 3; ++k) S[k] = -Sf_out[3 * i + k];", "for (int k = 0; k < 3; ++k) S[k] = Sf_out[3 * i + k];"),
 ("double lim = 0.05 * magd;", "double lim = 0.5 * magd;"),
 ("return (r < c->tolerance) || (c->rel_tol > 1e-20 && r < c->rel_tol * init);", "return (r < c->tolerance);"),

 ("diag[P] += gms * (-bdelta[i]);                   /* internalCoeffs", "diag[P] += gms * (-0.5*bdelta[i]);                   /* internalCoeffs"),
 ("gf = weights[f] * (gamma[owner[f]] - gamma[neighbour[f]]) + gamma[neighbour[f]];", "gf = weights[f] * (gamma[neighbour[f]] - gamma[owner[f]]) + gamma[owner[f]];"),
 ("if (fabs(wApA) / normFactor < 1e-300) {", "if (fabs(wApA) / normFactor < -1.0) {"),
 ("for (int c = 0; c < D[p].n_cells; ++c) W[p].rD[c] = 1.0 / D[p].diag[c];", "for (int c = 0; c < D[p].n_cells; ++c) W[p].rD[c] = 1.0;"),
 ("delta[i] = 1.0 / (nh[0] * e[0] + nh[1] * e[1] + nh[2] * e[2]);", "delta[i] = 1.0 / (nh[0] * e[0] + nh[1] * e[1] + nh[2] * e[2]) / 2;"),
 ("out[neighbour[f]] -= phi[f];", "out[neighbour[f]] += phi[f];"),
 ("if (bkind[b] != OR_EMPTY) out[bcells[b]] += bphi[b];", "out[bcells[b]] += bphi[b];"),
 ("for (int f = 0; f < n_faces; ++f) flux[f] = upper[f] * psi[neighbour[f]] - lower[f] * psi[owner[f]];", "for (int f = 0; f < n_faces; ++f) flux[f] = upper[f] * psi[owner[f]] - lower[f] * psi[neighbour[f]];"),
 ("bflux[b] = (gms * (-bdelta[b])) * psi[P] - ((-gms) * (bdelta[b] * bvalue[b]));", "bflux[b] = (gms * (-bdelta[b])) * psi[P] + ((-gms) * (bdelta[b] * bvalue[b]));"),
 # O11 GAMG
 ("if (ftc[o] < 0 && w[f] > bw) {", "if (ftc[o] < 0 && w[f] < bw + 1e300) {"),
 ("ftc[c] = best >= 0 ? ftc[best] : nc++;", "ftc[c] = nc++;"),
 ("else cdiag[ftc[owner[f]]] += upper[f] + upper[f];", "else cdiag[ftc[owner[f]]] += upper[f];"),
 ("if (frestrict[f] >= 0) cupper[frestrict[f]] += upper[f];", "if (frestrict[f] >= 0) cupper[frestrict[f]] = upper[f];"),
 ("for (int i = 0; i < n; ++i) coarse[ftc[i]] += fine[i];", "for (int i = 0; i < n; ++i) coarse[ftc[i]] = fine[i];"),
 ("L->x[i] = L->x[i] + omega * (L->rD[i] * (L->b[i] - L->y[i]));", "L->x[i] = L->x[i] + omega * (L->b[i] - L->y[i]);"),
 ("double a = fabs(den) > 1e-300 ? num / den : 1.0;", "double a = fabs(den) > 1e-300 ? den / num : 1.0;"),
 ("if (a < 0.0) a = 0.0;", "if (a < -10.0) a = 0.0;"),
 ("for (int i = 0; i < L->n; ++i) L->c[i] = Lv[l + 1].x[L->ftc[i]];", "for (int i = 0; i < L->n; ++i) L->c[i] = Lv[l + 1].x[L->ftc[i] / 2];"),
 ("for (int s = 0; s < gp->n_pre; ++s) or_smooth(L, gp);", ";"),
 ("for (int i = 0; i < L->n; ++i) L->r[i] = L->b[i] - L->y[i];", "for (int i = 0; i < L->n; ++i) L->r[i] = L->b[i];"),
 ("cw[l] += w[f];", "cw[l] = w[f];"),
 ("for (int i = 0; i < n; ++i) psi[i] = psi[i] + Lv[0].x[i];", "for (int i = 0; i < n; ++i) psi[i] = psi[i] - Lv[0].x[i];"),
 ("for (int f = 0; f < L->F; ++f) t[L->neighbour[f]] -= L->upper[f] * z[L->owner[f]];", "for (int f = 0; f < L->F; ++f) t[L->owner[f]] -= L->upper[f] * z[L->neighbour[f]];"),
 ("for (int i = 0; i < L->n; ++i) z[i] = L->rD[i] * t[i];", "for (int i = 0; i < L->n; ++i) z[i] = t[i];"),
 ("    if (gp->smoother == 1) or_gs2_sweep(L, gp->n_inner);", "    if (gp->smoother == 1) or_gs2_sweep(L, gp->n_inner > 0 ? gp->n_inner - 1 : 0);"),
 # O12 preconditioners / PBiCG / CSR
 ("for (int f = 0; f < F; ++f) rD[neighbour[f]] -= upper[f] * lower[f] / rD[owner[f]];", "for (int f = 0; f < F; ++f) rD[neighbour[f]] -= upper[f] * lower[f] / rD[neighbour[f]];"),
 ("    for (int c = 0; c < n; ++c) rD[c] = 1.0 / rD[c];\n}", "    ;\n}"),
 ("for (int f = 0; f < F; ++f) w[neighbour[f]] -= rD[neighbour[f]] * lo[f] * w[owner[f]];", "for (int f = 0; f < F; ++f) w[neighbour[f]] -= rD[neighbour[f]] * up[f] * w[owner[f]];"),
 ("for (int f = F - 1; f >= 0; --f) w[owner[f]] -= rD[owner[f]] * up[f] * w[neighbour[f]];\n        return;", "for (int f = 0; f < F; ++f) w[owner[f]] -= rD[owner[f]] * up[f] * w[neighbour[f]];\n        return;"),
 ("w[neighbour[f]] -= rD[neighbour[f]] * lo[f] * prev[owner[f]];", "w[neighbour[f]] -= rD[neighbour[f]] * lo[f] * w[owner[f]];"),
 ("                rT[c] -= alpha * wT[c];", "                rT[c] -= alpha * wA[c];"),
 ("or_pc_apply(kind, k, n, F, owner, neighbour, rD, upper, lower, rT, wT, 1);", "or_pc_apply(kind, k, n, F, owner, neighbour, rD, upper, lower, rT, wT, 0);"),
 ("    or_amul(n, F, owner, neighbour, diag, upper, lower, x, 0, 0, 0, 0, y); /* or_amul(diag, lower, upper): swapped */", "    or_amul(n, F, owner, neighbour, diag, lower, upper, x, 0, 0, 0, 0, y);"),
 ("t[3 * m + 2] = n + F + f;", "t[3 * m + 2] = n + f;"),
 ("        sumA[owner[f]] += upper[f];\n        sumA[neighbour[f]] += lower[f];", "        sumA[owner[f]] += lower[f];\n        sumA[neighbour[f]] += upper[f];"),
]
sel = os.environ.get("MUT_SELECT")  # e.g. "GAMG": only mutants after that marker
if sel == "GAMG":
    muts = muts[[a for a, _ in muts].index("if (ftc[o] < 0 && w[f] > bw) {"):]
elif sel == "O12":
    muts = muts[[a for a, _ in muts].index("for (int f = 0; f < F; ++f) rD[neighbour[f]] -= upper[f] * lower[f] / rD[owner[f]];"):]
res = []
for a, b in muts:
    assert a in src, a
try:
  for a, b in muts:
      assert a in src, a
      open('oracle/oracle.c', 'w').write(src.replace(a, b))
      import glob
      oracle_tests = sorted(glob.glob('tests/test_oracle_*.py')) + ['tests/test_multirank_gloo.py']
      r = subprocess.run([sys.executable, '-m', 'pytest', *oracle_tests, '-x', '-q', '-m', 'not gpu'], capture_output=True, text=True)
      caught = r.returncode != 0
      line = [l for l in r.stdout.splitlines() if l.startswith('FAILED')][:1]
      res.append((caught, a[:60], line))
      print(caught, a[:70], line, flush=True)
finally:
    open('oracle/oracle.c', 'w').write(src)
print('ALL CAUGHT' if all(c for c, *_ in res) else 'SOME MISSED')
