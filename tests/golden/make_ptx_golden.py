"""Golden outcomes of the REFERENCE PTX front-end on hand-written edge cases and
seeded random mutations of synthetic kernels (pins the native tokenizer
`libgkhost` and this package's `ptx.parse_ptx`).

Run in the build container only (imports /root/reference):

    python tests/golden/make_ptx_golden.py

Writes tests/golden/ptx_cases.json: per case the input (text, kernel, loop
counts, strict) and the reference outcome -- either the exception type and
message of `gpukalc.parse_ptx` / the pack step (KernelGraph.topo_order /
loop_multipliers), or the digest of the packed corpus of the reference graph.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path[:0] = [str(REF / "src"), str(ROOT), str(ROOT / "tests")]

import gpukalc as R  # noqa: E402

from goldens import corpus_digest  # noqa: E402
from paper_2305_01886_b200 import corpus as CG  # noqa: E402
from paper_2305_01886_b200 import pack  # noqa: E402

HEAD = ".version 7.0\n.target sm_70\n.address_size 64\n\n"


def k(body: str, name: str = "k") -> str:
    return HEAD + f".visible .entry {name}(\n\t.param .u64 p0\n)\n{{\n{body}\n}}\n"


EDGE = [
    ("empty_body", k(""), "k", {}),
    ("only_label", k("L0:"), "k", {}),
    ("missing_kernel", k("ret;"), "other", {}),
    ("no_entries", "// nothing here\n", "k", {}),
    ("unbalanced", HEAD + ".visible .entry k()\n{\n add.s32 %r1, %r2, %r3;\n", "k", {}),
    ("no_brace", HEAD + ".visible .entry k()\n", "k", {}),
    ("missing_semicolon", k("\tadd.s32 %r1, %r2, %r3\n\tret;"), "k", {}),
    ("unparseable", k("\t9add %r1;\n\tret;"), "k", {}),
    ("bad_head", k("\tadd-s32 %r1;\n"), "k", {}),
    ("unknown_label", k("\tbra NOWHERE;\n"), "k", {}),
    ("empty_branch", k("\tbra;\n"), "k", {}),
    ("duplicate_label", k("A:\n\tadd.s32 %r1, %r1, 1;\nA:\n\tret;"), "k", {}),
    ("auto_label_clash", k("\tadd.s32 %r1, %r1, 1;\nbra_t:\nbb0:\n\tret;"), "k", {}),
    ("loop_ok", k("L:\n\tadd.s32 %r1, %r1, 1;\n\tsetp.lt.s32 %p1, %r1, 8;\n"
                  "\t@%p1 bra L;\n\tret;"), "k", {"L": 8}),
    ("loop_missing_count", k("L:\n\tadd.s32 %r1, %r1, 1;\n\t@%p1 bra L;\n\tret;"), "k", {}),
    ("loop_bad_label", k("L:\n\tadd.s32 %r1, %r1, 1;\n\t@%p1 bra L;\n\tret;"), "k",
     {"L": 3, "Q": 2, "A": 1}),
    ("loop_two_back_edges", k("L:\n\tadd.s32 %r1, %r1, 1;\n\t@%p1 bra L;\n"
                              "\tadd.s32 %r2, %r2, 1;\n\t@%p2 bra L;\n\tret;"), "k", {"L": 4}),
    ("nested_loops", k("A:\n\tadd.s32 %r1, %r1, 1;\nB:\n\tmul.lo.s32 %r2, %r2, 3;\n"
                       "\t@%p1 bra B;\n\t@%p2 bra A;\n\tret;"), "k", {"A": 5, "B": 7}),
    ("mult_overflow", k("A:\n\tadd.s32 %r1, %r1, 1;\nB:\n\tmul.lo.s32 %r2, %r2, 3;\n"
                        "\t@%p1 bra B;\n\t@%p2 bra A;\n\tret;"), "k",
     {"A": 4_000_000_000, "B": 4_000_000_000}),
    ("mult_zero", k("A:\n\tadd.s32 %r1, %r1, 1;\n\t@%p2 bra A;\n\tret;"), "k", {"A": 0}),
    ("mult_negative", k("A:\n\tadd.s32 %r1, %r1, 1;\n\t@%p2 bra A;\n\tret;"), "k", {"A": -3}),
    ("self_loop_uncond", k("A:\n\tadd.s32 %r1, %r1, 1;\n\tbra A;\n"), "k", {"A": 2}),
    ("pred_fallthrough_dup", k("\t@%p1 bra N;\nN:\n\tret;"), "k", {}),
    ("pred_ret", k("\t@%p1 ret;\n\tadd.s32 %r1, %r1, 1;\n\texit;\n\tmov.u32 %r2, %r1;"), "k", {}),
    ("comments", k("/* a\n b */ add.s32 %r1, %r2, %r3; // c\n\t// ld.global.f32 %f1, [%rd1];\n"
                   "\tmul.f32 %f1, %f2, %f3; /* x */ ret;"), "k", {}),
    ("comment_spans_lines", k("\tadd.s32 %r1, %r2, %r3; // x /* y\n\tmul.lo.s32 %r4, %r1, 2;\n"
                              "\t*/ sub.s32 %r5, %r4, %r1;\n\tret;"), "k", {}),
    ("unclosed_block_comment", k("\tadd.s32 %r1, %r2, %r3;\n\t/* never closed\n\tret;"), "k", {}),
    ("crlf", k("\tadd.s32 %r1, %r2, %r3;\r\n\tret;\r\n").replace("\n", "\r\n"), "k", {}),
    ("many_per_line", k("A: add.s32 %r1, %r2, %r3; B: mul.lo.s32 %r4, %r1, %r1; bra A;"), "k",
     {"A": 3}),
    ("directives_braces", k("\t.reg .b32 %r<9>;\n\t{\n\t.reg .pred %p<3>;\n\tadd.s32 %r1, %r2, 1;\n"
                            "\t}\n\tret;"), "k", {}),
    ("vectors_special", k("\tmov.u32 %r1, %tid.x;\n\tmov.u32 %ctaid.y, %r1;\n"
                          "\tld.global.v2.f32 {%f1, %f2}, [%rd1+8];\n"
                          "\tst.global.v2.f32 [%rd2], {%f1, %f2};\n\tadd.f32 %f3, %f1, %f2;\n"
                          "\tmov.b64 %rd3, {%r1.x, %r1.y};\n\tret;"), "k", {}),
    ("bracket_dest", k("\tatom.global.add.u32 [%rd1], %r1;\n\tld.shared.f32 %f1, [%r2];\n"
                       "\tst.shared.f32 [%r2+4], %f1;\n\tred.global.add.u32 [%rd1], %r3;\n\tret;"),
     "k", {}),
    ("f64_dpu", k("\tadd.f64 %fd1, %fd2, %fd3;\n\tdiv.rn.f64 %fd4, %fd1, %fd2;\n"
                  "\tsqrt.rn.f64 %fd5, %fd4;\n\tfma.rn.f64 %fd6, %fd5, %fd1, %fd2;\n\tret;"), "k", {}),
    ("unknown_opcode", k("\tfrobnicate.b32 %r1, %r2;\n\tadd.s32 %r3, %r1, 1;\n\tret;"), "k", {}),
    ("unknown_opcode_strict", k("\tfrobnicate.b32 %r1, %r2;\n\tret;"), "k", {}, True),
    ("generic_and_spaces", k("\tld.f32 %f1, [%rd1];\n\tld..f32 %f2, [%rd1];\n"
                             "\tld.param.u64 %rd2, [p0];\n\tld.const.f32 %f3, [c];\n"
                             "\tld.local.f32 %f4, [l];\n\tldu.global.f32 %f5, [%rd1];\n"
                             "\tprefetch.global.L1 [%rd1];\n\tret;"), "k", {}),
    ("pred_no_space", k("\t@%p1bra L;\nL:\n\tret;"), "k", {}),
    ("pred_neg_spaces", k("\t@!%p1   \t bra L;\n\tadd.s32 %r1, %r1, 1;\nL:\n\tret;"), "k", {}),
    ("ops_empty_middle", k("\tadd.s32 %r1, , %r2;\n\tadd.s32 %r3,%r1,%r1 ;\n\tret;"), "k", {}),
    ("unicode_free_dollar", k("$L__BB0_1:\n\tadd.s32 %r$1, %r$2, 1;\n\tbra.uni $L__BB0_1;\n"),
     "k", {"$L__BB0_1": 2}),
    ("two_kernels_second",
     HEAD + ".visible .entry a()\n{\n\tret;\n}\n.visible .entry b()\n{\n\tadd.s32 %r1, %r1, 1;\n"
     "\tret;\n}\n", "b", {}),
    ("entry_tab_name", HEAD + ".entry\tk2()\n{\n\tret;\n}\n", "k2", {}),
    ("entry_no_space", HEAD + ".entryk()\n{\n\tret;\n}\n", "k", {}),
    ("label_then_directive", k("A: .reg .b32 %r<2>;\n\tret;"), "k", {}),
    ("semicolons_only", k(";;;\n\tret;"), "k", {}),
    ("brace_lines", k("{ add.s32 %r1, %r1, 1; }\n\tret;"), "k", {}),
    ("call_and_bar", k("\tcall.uni (%r1), f, (%r2);\n\tbar.sync 0;\n\tmembar.gl;\n\tret;"), "k", {}),
]

NOISE = [";", "}", "{", "//", "/*", "*/", "@%p1 ", "@!%p9 ", "bra L1;", "bra $X;", "LBL:", "L1:",
         ".reg .b32 %r<4>;", "\r", "\t", " ", "\n", "foo.bar %r1;", "@!%p2 bra L1;", "ret;",
         "exit;", "ld.global.v2.f32 {%f1, %f2}, [%rd1+4];", "%", ",", "[", "]", "9", ".",
         "add.f64 %fd1, %fd1, %fd2;", "st.global.f32 [%rd1], %f1;", "bar.sync 0;"]


def mutate(rng: random.Random, text: str) -> str:
    for _ in range(rng.randint(1, 4)):
        op = rng.random()
        if not text:
            break
        i = rng.randrange(len(text))
        if op < 0.3:
            text = text[:i] + text[i + rng.randint(1, 8):]
        elif op < 0.7:
            text = text[:i] + rng.choice(NOISE) + text[i:]
        else:
            lines = text.split("\n")
            j = rng.randrange(len(lines))
            if rng.random() < 0.5:
                del lines[j]
            else:
                lines.insert(j, lines[rng.randrange(len(lines))])
            text = "\n".join(lines)
    return text


def outcome(text: str, name: str, loops: dict, strict: bool) -> dict:
    try:
        g = R.parse_ptx(text, name, loop_counts=loops, strict_opcodes=strict)
        c = pack.pack_corpus([g])  # topo_order / loop_multipliers of the reference graph
    except Exception as exc:  # noqa: BLE001 - the outcome IS the exception
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"digest": corpus_digest(c), "n_tok": int(c.n_tok), "n_blk": int(len(c.blk))}


def main() -> None:
    cases = []
    for e in EDGE:
        name, text, kern, loops = e[:4]
        strict = bool(e[4]) if len(e) > 4 else False
        cases.append({"name": name, "text": text, "kernel": kern, "loops": loops, "strict": strict,
                      "ref": outcome(text, kern, loops, strict)})
    rng = random.Random(20261017)
    for i, (kname, text, loops) in enumerate(CG.synth_corpus(250, 77)):
        t = mutate(rng, text)
        lp = dict(loops)
        r = rng.random()
        if r < 0.1 and lp:
            lp.pop(next(iter(lp)))
        elif r < 0.15:
            lp["NOT_A_LABEL"] = 3
        cases.append({"name": f"mut{i}", "text": t, "kernel": kname, "loops": lp, "strict": False,
                      "ref": outcome(t, kname, lp, False)})
    (HERE / "ptx_cases.json").write_text(json.dumps({"source": "gpukalc (reference) parse_ptx",
                                                      "cases": cases}))
    kinds: dict = {}
    for c in cases:
        key = c["ref"].get("error", "ok")
        kinds[key] = kinds.get(key, 0) + 1
    print(len(cases), "cases", kinds)


if __name__ == "__main__":
    main()
