#!/bin/bash
# Mutation check of the oracle pins: each line injects one plausible mistake into
# oracle/oracle.c and expects tests/test_oracle_pins.py to FAIL.  Restores the file.
# Run from the repo root:  bash tools/oracle_mutation_check.sh
set -u
cd "$(dirname "$0")/.."
mut() {  # mut SED NAME [TESTFILE]
  cp oracle/oracle.c /tmp/oracle.c.bak
  sed -i "$1" oracle/oracle.c
  if cmp -s oracle/oracle.c /tmp/oracle.c.bak; then echo "[$2] SED DID NOT APPLY"; return; fi
  rm -f oracle/liboracle.so
  r=$(timeout 600 python -m pytest "${3:-tests/test_oracle_pins.py}" -x -q 2>&1 | tail -1)
  echo "[$2] $r"
  cp /tmp/oracle.c.bak oracle/oracle.c
  rm -f oracle/liboracle.so
}
mut 's/(i128)st->deg\[own\] - di)/(i128)st->deg[own])/' "drop -delta_i in S_own (Eq.4 C(i)\\{i})"
mut 's/(S == S_best \&\& c < best)/(S == S_best \&\& c > best)/' "max-label tie (P:L95)"
mut 's/best >= 0 \&\& S_best > S_own/best >= 0 \&\& S_best >= S_own/' "non-strict move (P:L223)"
mut 's/st->size\[best\] == 1 \&\& best > own) result = own;/st->size[best] == 1 \&\& best < own) result = own;/' "singlet rule inverted (P:L92)"
mut 's/int64_t s = 2 \* g->loop\[i\];/int64_t s = g->loop[i];/' "loop once in delta (D2)"
mut 's/s += 2 \* g->loop\[i\];/s += g->loop[i];/' "loop once in I2 (D24)"
mut 's/h->loop\[c\] += intra2\[c\] \/ 2;/h->loop[c] += intra2[c];/' "induce double intra (D19)"
mut 's/id\[c\] = used\[c\] ? (int32_t)k++ : -1;/id[c] = used[c] ? (int32_t)(k++) : -1; if (used[c] \&\& k > 1) id[c] = (int32_t)(k - 1) ^ 1;/' "renumber not order-preserving (D18)"
mut 's/if (mode == 1 \&\& st->size\[own\] != 1) return own;/if (0) return own;/' "merge non-singlets (D14)"
mut 's/st->deg\[labels\[i\]\] += g->delta\[i\];/st->deg[labels[i]] += 1;/' "deg as count (Eq.2)"
mut 's/i128 S = twoW \* sc->e\[c\] - di \* (i128)st->deg\[c\];/i128 S = twoW * sc->e[c] + di * (i128)st->deg[c];/' "sign flip in S (Eq.4)"
mut 's/if (out > 0 \&\& buf\[out - 1\].v == buf\[k\].v) buf\[out - 1\].w += buf\[k\].w;/if (out > 0 \&\& buf[out - 1].v == buf[k].v) buf[out - 1].w = buf[k].w;/' "duplicates not summed (D25)"
mut 's/for (int64_t t = 0; t < nt; ++t) { sc->e\[sc->touched\[t\]\] = 0; sc->mark\[sc->touched\[t\]\] = 0; }/for (int64_t t = 0; t < nt; ++t) { sc->mark[sc->touched[t]] = 0; }/' "Eq.1 scratch not reset between vertices"
mut 's/for (s = 1; s <= cfg->max_sweeps; ++s) {/for (s = 1; s <= cfg->max_sweeps - 1; ++s) {/' "cap off by one (D12)"
mut 's/if (l == 0 || !(Ql - mod_curr < cfg->big_theta))/if (!(Ql - mod_curr < cfg->big_theta))/' "level 0 not forced (Alg.2)"
mut 's/return neg ? -d : d;/return d;/' "d128 sign lost (D22)"
# real weights (F1, reading D28) -> tests/test_oracle_real.py
R=tests/test_oracle_real.py
mut 's/static double fixed_of(double w, int32_t s) { return rint(ldexp(w, s)); }/static double fixed_of(double w, int32_t s) { return round(ldexp(w, s)); }/' "half away from zero (D28 rint)" $R
mut 's/if (og_fixed_sum(m, w, mid) <= lim) lo = mid; else hi = mid;/if (og_fixed_sum(m, w, mid) < lim \/ 2) lo = mid; else hi = mid;/' "scale one bit short (D28 largest s)" $R
mut 's/const int64_t lim = (int64_t)1 << 52;/const int64_t lim = (int64_t)1 << 53;/' "2W budget instead of W (D28)" $R
mut 's/int32_t lo = -1100, hi = 1100; /int32_t lo = -60, hi = 60; /' "scale search range too narrow (D28)" $R
# colouring heuristic (F2, reading D29) -> tests/test_oracle_coloring.py
Cf=tests/test_oracle_coloring.py
mut 's/return x < y ? 1 : x > y ? -1 : 0;/return x < y ? -1 : x > y ? 1 : 0;/' "ascending priority order (D29)" $Cf
mut 's/k ^= k >> 33; k \*= 0xff51afd7ed558ccdull;/k ^= k >> 31; k *= 0xff51afd7ed558ccdull;/' "wrong fmix64 shift (D29)" $Cf
mut 's/while (used\[c\]) ++c;                                              \/\* smallest free \*\//c = 0; while (used[c]) c += 2;/' "not the smallest free colour (D29)" $Cf
mut 's/memcpy(cur, labels_out, (size_t)n \* sizeof(int32_t));   \/\* commit class c \*\//(void)0;/' "classes see the sweep-start state (Jacobi, D29)" $Cf
