"""The R-block record permutations (paper_2605_19660_b200/csrc/layout.h) are
bijections: every (token, channel) code of a block lands in exactly one field of
one word, every (channel, group) / (token, group) parameter in exactly one slot,
every token norm in one slot -- for INT2, INT4 and the bf16 record.  Compiled
host-side from the same header the kernels use (no GPU needed)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROGRAM = r"""
#include <cstdio>
#include <vector>
#include "layout.h"
using namespace osk;

static int check_codes(int bits) {
    const int tpw = 16 / bits, nwords = R * D * bits / 32;
    std::vector<int> seen_k(R * D, 0), seen_v(R * D, 0);
    for (int w = 0; w < nwords; ++w)
        for (int hi = 0; hi < 2; ++hi)
            for (int f = 0; f < tpw; ++f) {
                int t, c;
                k_word_coords(bits, w, f, hi, t, c);
                if (t < 0 || t >= R || c < 0 || c >= D) return 1;
                seen_k[t * D + c]++;
                v_word_coords(bits, w, f, hi, t, c);
                if (t < 0 || t >= R || c < 0 || c >= D) return 2;
                seen_v[t * D + c]++;
            }
    for (int i = 0; i < R * D; ++i)
        if (seen_k[i] != 1 || seen_v[i] != 1) return 3;
    return 0;
}

static int check_params() {
    std::vector<int> ka(D * NGRP, 0), kb(D * NGRP, 0), va(R * NGC, 0), vb(R * NGC, 0), nr(R, 0);
    for (int c = 0; c < D; ++c)
        for (int g = 0; g < NGRP; ++g) {
            const int a = ka_index(c, g), b = kb_index(c, g);
            if (a < 0 || a >= D * NGRP || b < 0 || b >= D * NGRP) return 10;
            ka[a]++;
            kb[b]++;
        }
    for (int t = 0; t < R; ++t) {
        for (int g = 0; g < NGC; ++g) {
            const int a = va_index(t, g), b = vb_index(t, g);
            if (a < 0 || a >= R * NGC || b < 0 || b >= R * NGC) return 11;
            va[a]++;
            vb[b]++;
        }
        const int n = norm_index(t);
        if (n < 0 || n >= R) return 12;
        nr[n]++;
    }
    for (int i = 0; i < D * NGRP; ++i)
        if (ka[i] != 1 || kb[i] != 1) return 13;
    for (int i = 0; i < R * NGC; ++i)
        if (va[i] != 1 || vb[i] != 1) return 14;
    for (int i = 0; i < R; ++i)
        if (nr[i] != 1) return 15;
    return 0;
}

static int check_bf16() {
    // one 32-token quarter: 4096 words of K and of V, two bf16 each
    std::vector<int> sk(32 * D, 0), sv(32 * D, 0);
    for (int w = 0; w < 32 * D / 2; ++w)
        for (int hi = 0; hi < 2; ++hi) {
            int t, c;
            bf16_k_coords(w, hi, t, c);
            if (t < 0 || t >= 32 || c < 0 || c >= D) return 20;
            sk[t * D + c]++;
            bf16_v_coords(w, hi, t, c);
            if (t < 0 || t >= 32 || c < 0 || c >= D) return 21;
            sv[t * D + c]++;
        }
    for (int i = 0; i < 32 * D; ++i)
        if (sk[i] != 1 || sv[i] != 1) return 22;
    return 0;
}

// the inverse maps the per-element readers (logits kernel) use
static int check_inverse(int bits) {
    const int tpw = 16 / bits, nwords = R * D * bits / 32;
    for (int w = 0; w < nwords; ++w)
        for (int hi = 0; hi < 2; ++hi)
            for (int f = 0; f < tpw; ++f) {
                int t, c, w2, s2;
                k_word_coords(bits, w, f, hi, t, c);
                k_code_loc(bits, t, c, w2, s2);
                if (w2 != w || s2 != hi * 16 + f * bits) return 30;
                v_word_coords(bits, w, f, hi, t, c);
                v_code_loc(bits, t, c, w2, s2);
                if (w2 != w || s2 != hi * 16 + f * bits) return 31;
            }
    for (int qu = 0; qu < 4; ++qu)
        for (int w = 0; w < 32 * D / 2; ++w)
            for (int hi = 0; hi < 2; ++hi) {
                int t, c;
                bf16_k_coords(w, hi, t, c);
                if (bf16_k_byte(qu * 32 + t, c) != qu * BF16_QUARTER_BYTES + w * 4 + hi * 2) return 32;
            }
    return 0;
}

int main() {
    int rc = check_codes(2);
    if (!rc) rc = check_codes(4);
    if (!rc) rc = check_params();
    if (!rc) rc = check_bf16();
    if (!rc) rc = check_inverse(2);
    if (!rc) rc = check_inverse(4);
    std::printf("layout rc %d\n", rc);
    return rc;
}
"""


def test_record_permutations_are_bijections(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "layout_check.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "layout_check"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "paper_2605_19660_b200", "csrc"),
                    str(src), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
