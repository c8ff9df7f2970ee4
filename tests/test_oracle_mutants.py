"""Mutation check of the oracle's pins ("removing any flush must
break equivalence"): each plausible mistake below -- a dropped term, a
wrong sign or index, a transposed layout, a swapped order, an off-by-one in
the item split -- is compiled into a copy of oracle/escs_oracle.c, and
tests/test_oracle.py (the pins: dense numpy, exact dyadic, identities, golden
plans, exhaustive patterns, brute force, invariants) must FAIL against it.
A surviving mutant is a gap in the pins."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "escs_oracle.c")

MUTANTS = [
    # oracle_spmm (Listing 1)
    ("spmm: first term of every row dropped",
     "for (int64_t t = rowptr[i]; t < rowptr[i + 1]; t++) {",
     "for (int64_t t = rowptr[i] + 1; t < rowptr[i + 1]; t++) {"),
    ("spmm: last term of every row dropped",
     "for (int64_t t = rowptr[i]; t < rowptr[i + 1]; t++) {",
     "for (int64_t t = rowptr[i]; t < rowptr[i + 1] - 1; t++) {"),
    ("spmm: sign of A dropped",
     "c[j] += av * (double)b[j];",
     "c[j] += fabs(av) * (double)b[j];"),
    ("spmm: B row indexed by the output row (transposed operand)",
     "const float *b = B + kk * (int64_t)ncols;",
     "const float *b = B + (i % k) * (int64_t)ncols;"),
    ("spmm: B column index reversed",
     "c[j] += av * (double)b[j];",
     "c[j] += av * (double)b[ncols - 1 - j];"),
    ("spmm: fp32 accumulation",
     "c[j] += av * (double)b[j];",
     "c[j] = (double)(float)(c[j] + av * (double)b[j]);"),
    # oracle_partition (dataTransformer P:575-577, Fig. 4, Listing 7 / Reading R1, R7)
    ("partition: pattern bits in reversed row order",
     "mask[colidx[t]] |= (int32_t)1 << r;",
     "mask[colidx[t]] |= (int32_t)1 << (h - 1 - r);"),
    ("partition: groups in descending pattern order",
     "for (int64_t mu = 1; mu < nmask; mu++) {\n            if (count[mu] == 0) continue;",
     "for (int64_t mu = nmask - 1; mu >= 1; mu--) {\n            if (count[mu] == 0) continue;"),
    ("partition: value slots row-major instead of column-major (R1)",
     "slot_src[grp_val_ptr[g] + ci * p + rank] = pos[(int64_t)r * k + c];",
     "slot_src[grp_val_ptr[g] + rank * count[mu] + ci] = pos[(int64_t)r * k + c];"),
    ("partition: value slot of the wrong pattern row",
     "slot_src[grp_val_ptr[g] + ci * p + rank] = pos[(int64_t)r * k + c];",
     "slot_src[grp_val_ptr[g] + ci * p + (p - 1 - rank)] = pos[(int64_t)r * k + c];"),
    ("partition: NPP advanced by width instead of popcount x width",
     "grp_val_ptr[NG + 1] = (int32_t)(grp_val_ptr[NG] + count[mu] * p);",
     "grp_val_ptr[NG + 1] = (int32_t)(grp_val_ptr[NG] + count[mu] * p - (p > 1));"),
    ("partition: item count floor instead of ceil",
     "int64_t nPi = (SP + T - 1) / T;",
     "int64_t nPi = SP / T;"),
    ("partition: item boundary rounding",
     "int64_t s0 = (q * SP) / nPi, s1 = ((q + 1) * SP) / nPi;",
     "int64_t s0 = (q * SP + nPi - 1) / nPi, s1 = ((q + 1) * SP + nPi - 1) / nPi;"),
    ("partition: item_group_begin takes the first group starting after s0",
     "if (grp_col_ptr[g] - pstream0 <= s0) gb = g;",
     "if (grp_col_ptr[g] - pstream0 < s0) gb = g;"),
    ("partition: panel image not reset between panels",
     "for (int64_t c = 0; c < k; c++) mask[c] = 0;",
     "for (int64_t c = 0; c < 0; c++) mask[c] = 0;"),
]


@pytest.mark.parametrize("name,old,new", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_pins_kill_mutant(tmp_path, name, old, new):
    src = open(SRC).read()
    assert src.count(old) == 1, f"mutation site not unique: {old!r}"
    mut = tmp_path / "mutant.c"
    mut.write_text(src.replace(old, new))
    lib = tmp_path / "libmutant.so"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o",
                           str(lib), str(mut), "-lm"])
    env = dict(os.environ, ESCS_ORACLE_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant survived the oracle pins: {name}\n{r.stdout[-2000:]}"


def test_control_unmutated_copy_passes(tmp_path):
    """The same harness on an unmodified copy passes (so a kill above is the
    mutation's doing, not the harness's)."""
    lib = tmp_path / "libcontrol.so"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o",
                           str(lib), SRC, "-lm"])
    env = dict(os.environ, ESCS_ORACLE_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]
