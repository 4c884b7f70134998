"""Mutation check of the oracle pins (-m "not gpu").

Each case rebuilds ``oracle/turbo_oracle.c`` with one plausible misreading
planted (the ones a decode or quantiser could share with a kernel written from
the same reading) and requires the CPU pin suite to FAIL on it.  A mutation the
pins let through would mean the oracle is not pinned against that mistake.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "turbo_oracle.c")
PINS = ["tests/test_oracle_decode_pins.py", "tests/test_oracle_pins.py", "tests/test_chunked_oracle.py",
        "tests/test_oracle_sas_fp16.py"]

# (name, original text, mutated text) -- each original must occur in the source
MUTATIONS = [
    ("V parent scale from the K slot (P:970)",
     "s_v = is_buf ? st1(p, vs->a_univ / TQ_DIV) : vs->s_parent[j];",
     "s_v = is_buf ? st1(p, vs->a_univ / TQ_DIV) : ks->s_parent[j];"),
    ("buffer K scale not a_univ/119 (P:451-453)",
     "s_k = is_buf ? st1(p, ks->a_univ / TQ_DIV) : ks->s_parent[j];",
     "s_k = is_buf ? st1(p, ks->a_univ / 127.0f) : ks->s_parent[j];"),
    ("buffer V codes read from the K slot",
     "vh[ie] = vs->buf[ie];",
     "vh[ie] = ks->buf[ie];"),
    ("V dequantised without the zero point (P:966-967)",
     "vh[ie] = (int8_t)tq_dequant_q2(vs->codes[cb], vs->s_int[sb], vs->z_int[sb]);",
     "vh[ie] = (int8_t)tq_dequant_q2(vs->codes[cb], vs->s_int[sb], 0);"),
    ("decode P scale kept across blocks (per split, not per row x block; P:977)",
     "sp = quant_p(nc, pt, &row_active, nc, pc);          /* per-row P scale (P:976-977, R-17) */",
     "{ static float keep = 0.0f; float mx = keep; for (int32_t c = 0; c < nc; ++c) mx = fmaxf(mx, pt[c]);"
     " keep = t + 1 < n_tiles ? mx : 0.0f; float tmp[1024]; memcpy(tmp, pt, sizeof(float) * nc); tmp[0] = "
     "fmaxf(tmp[0], mx); sp = quant_p(nc, tmp, &row_active, nc, pc); }"),
    ("decode alpha = 1 always",
     "row_step(p, nc, x, &m, &l, pt, &alpha);               /* P:972-974 */",
     "row_step(p, nc, x, &m, &l, pt, &alpha); if (t > 0) { l = l / alpha * 1.0; alpha = 1.0; }"),
    ("stage-1 codes round half away from zero (R-2)",
     "codes[i] = (int8_t)rint((double)x[i] * (double)inv);",
     "codes[i] = (int8_t)round((double)x[i] * (double)inv);"),
    ("stage-2 codes round half to even (R-6)",
     "codes[(int64_t)t * code_stride] = (uint8_t)((2 * (v - mn) + s) / (2 * s));",
     "codes[(int64_t)t * code_stride] = (uint8_t)rint((double)(v - mn) / s);"),
    ("prefill P scale per row instead of per B_r x B_c tile (P:918)",
     "sp = quant_p((int64_t)nr * nc, pt, active, nc, pc);",
     "for (int32_t r = 0; r < nr; ++r) sp = quant_p(nc, pt + (int64_t)r * nc, active + r, nc, pc + (int64_t)r * nc);"),
    ("FP16 scale variant: flushed-buffer parent scale left in FP32 (R-29)",
     "flush_block(p, s, s->buf, st1(p, s->a_univ / TQ_DIV));",
     "flush_block(p, s, s->buf, s->a_univ / TQ_DIV);"),
    ("FP16 scale variant: binary16 ties rounded away from zero (R-29)",
     "double r = ldexp(rint(ldexp(a, -q)), q);",
     "double r = ldexp(round(ldexp(a, -q)), q);"),
    ("FP16 SAS: fraction left in binary32 (R-30)",
     "const float fh = round_fp16(f);",
     "const float fh = f;"),
    ("FP16 SAS: binary16 FMA double-rounded through binary32 (R-30)",
     "  return fma_fp16(fma_fp16(fma_fp16(c3, fh, c2), fh, c1), fh, c0);",
     "  return round_fp16(fmaf(round_fp16(fmaf(round_fp16(fmaf(c3, fh, c2)), fh, c1)), fh, c0));"),
    ("FP16 SAS: Horner in binary32, rounded to binary16 once (R-30)",
     "  return fma_fp16(fma_fp16(fma_fp16(c3, fh, c2), fh, c1), fh, c0);",
     "  return round_fp16(fmaf(fmaf(fmaf(c3, fh, c2), fh, c1), fh, c0));"),
    ("FP16 SAS not used for alpha (R-30)",
     "  else alpha = (double)sas_p(p, m_new - m_prev);",
     "  else alpha = (double)tq_sas(m_new - m_prev, p->sas_nr);"),
    ("universal scale from the last block only (R-9)",
     "float a_univ = 0.0f;\n  for (int64_t i = 0; i < (int64_t)n * d; ++i) a_univ = fmaxf(a_univ, fabsf(x[i]));",
     "float a_univ = 0.0f;\n  for (int64_t i = (int64_t)(n - 1) / bc * bc * d; i < (int64_t)n * d; ++i)"
     " a_univ = fmaxf(a_univ, fabsf(x[i]));"),
]


@pytest.mark.parametrize("name,orig,mut", MUTATIONS, ids=[m[0] for m in MUTATIONS])
def test_pins_catch_mutation(tmp_path, name, orig, mut):
    src = open(SRC).read()
    assert src.count(orig) == 1, f"mutation anchor not found once: {orig!r}"
    msrc = tmp_path / "turbo_oracle.c"
    msrc.write_text(src.replace(orig, mut))
    lib = tmp_path / "libmut.so"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "oracle"), str(msrc), "-o", str(lib), "-lm"])
    env = dict(os.environ, TURBO_ORACLE_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *PINS],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0, f"pins passed with mutation '{name}':\n{r.stdout[-2000:]}"
