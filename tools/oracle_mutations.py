"""Mutation check of the oracle's pins: apply one plausible slip at a time to a
copy of oracle/starsd_ref.c, rebuild the copy, and run the CPU pin suites against it.  Every
mutation must make at least one pin fail.  Usage: python tools/oracle_mutations.py"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTATIONS = [
    ("accept_probs: a without min(1, .)", "a_out[j] = ell >= 0.0 ? 1.0 : exp(ell);", "a_out[j] = exp(ell);"),
    ("accept_probs: u from w1", "sd_ref_uniforms(seed, (uint32_t)j, round, rid_base + (uint64_t)b, &u_out[j], NULL);",
     "sd_ref_uniforms(seed, (uint32_t)j, round, rid_base + (uint64_t)b, NULL, &u_out[j]);"),
    ("trace: mu_s not divided by R", "tr->mu_s = (m1 < m2 ? m1 : m2) / R;", "tr->mu_s = (m1 < m2 ? m1 : m2);"),
    ("trace: mu_a against ell", "double mu = fabs(u_acc - acc);", "double mu = fabs(u_acc - ell);"),
    ("trace: C_prev = C(t)", "            *C_prev = C;\n            *C_tok = Cn;", "            *C_prev = Cn;\n            *C_tok = Cn;"),
    ("sample_check: C(t-1) includes t", "for (int32_t y = 0; y < t; ++y) C += buf[y];", "for (int32_t y = 0; y <= t; ++y) C += buf[y];"),
    ("sample_check: u_smp of position 0", "sd_ref_uniforms(seed, (uint32_t)L, round, rid_base + (uint64_t)b, NULL, &u_smp);",
     "sd_ref_uniforms(seed, 0u, round, rid_base + (uint64_t)b, NULL, &u_smp);"),
    ("sampling_dist: no C-6 fallback", "        if (R > 0.0) return R;\n        *zero_res = 1;", "        return R;\n        *zero_res = 1;"),
    ("sampling_dist: residual q - p", "double d = prob_of(pr, y, T, lam_p) - prob_of(*qr, y, T, lam_q);",
     "double d = prob_of(*qr, y, T, lam_q) - prob_of(pr, y, T, lam_p);"),
    ("tree: no residual between candidates (outcome)", "                if (i > 0) residual_step(pb, qb, V);\n                double acc = qb[x] > 0.0",
     "                double acc = qb[x] > 0.0"),
    ("tree: final sample from p, not d_m (walk)", "        /* every candidate rejected: t ~ d_m */\n        if (residual_step(pb, qb, V) == 0.0) status |= SD_REF_FAULT_ZERO_RESIDUAL;",
     "        /* every candidate rejected: t ~ d_m */"),
    ("tree: candidate counter without the 32 i stride", "sd_ref_uniforms(a->seed, (uint32_t)(depth + 32 * i), a->round, rid, &u, NULL);",
     "sd_ref_uniforms(a->seed, (uint32_t)(depth + i), a->round, rid, &u, NULL);"),
    ("verify: u_acc from w1", "sd_ref_uniforms(a->seed, (uint32_t)j, a->round, rid, &u_acc, NULL);",
     "sd_ref_uniforms(a->seed, (uint32_t)j, a->round, rid, NULL, &u_acc);"),
]
SUITES = ["tests/test_oracle_checkers.py", "tests/test_oracle_pins.py", "tests/test_oracle_tree.py"]


def main():
    src = open(os.path.join(ROOT, "oracle", "starsd_ref.c")).read()
    bad = 0
    for name, old, new in MUTATIONS:
        assert src.count(old) == 1, (name, src.count(old))
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "workload"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            open(os.path.join(tmp, "oracle", "starsd_ref.c"), "w").write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"]
                               + SUITES, cwd=tmp, capture_output=True, text=True)
            caught = r.returncode != 0
            bad += not caught
            last = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
            print(f"{'CAUGHT' if caught else 'MISSED'}  {name}  {last[0] if last else ''}", flush=True)
    print(f"{len(MUTATIONS) - bad}/{len(MUTATIONS)} mutations caught")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
