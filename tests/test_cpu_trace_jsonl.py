"""CPU: JSONL trace ingestion (cace_trace_parse_jsonl, csrc/trace_jsonl.hpp)
vs the reference's parse_trace (workload.cpp:204-266) compiled in oracle/_ref.

Parsed columns and headers must be identical; every ParseError the reference
raises must come back with the same text (JSON syntax errors: same
"trace line N: invalid JSON: " prefix)."""
import json

import numpy as np
import pytest

P = pytest.importorskip("paper_2506_18796_b200")
from paper_2506_18796_b200 import api  # noqa: E402


def _ours(text: bytes):
    return api.parse_trace(text, api.ModelCatalog.build_default())


def _same(ref, text: bytes):
    want = ref.parse_trace(text)
    tr, hdr, rid = _ours(text)
    assert (hdr.pattern, hdr.seed, hdr.windows) == (want["pattern"], want["seed"], want["windows"])
    assert np.float64(hdr.arrival_rate_per_s).view(np.uint64) == np.float64(want["rate"]).view(np.uint64)
    assert np.float64(hdr.window_duration_s).view(np.uint64) == np.float64(want["duration"]).view(np.uint64)
    assert np.array_equal(rid, want["request_id"])
    assert np.array_equal(tr.arrival_time_s.view(np.uint64), want["arrival"].view(np.uint64))
    assert np.array_equal(tr.prompt_tokens, want["prompt"]) and np.array_equal(tr.output_tokens, want["output"])
    cat = api.ModelCatalog.build_default()
    exp_model = np.array([cat.lookup(int(l), int(c)) for l, c in zip(want["language"], want["task_class"])],
                         np.int32)
    assert np.array_equal(tr.model, exp_model)
    return tr


def _err(ref, text: bytes, prefix_only=False):
    with pytest.raises(Exception) as e_ref:
        ref.parse_trace(text)
    with pytest.raises(api.SimError) as e_ours:
        _ours(text)
    a, b = str(e_ref.value), str(e_ours.value)
    if prefix_only:
        k = a.index("invalid JSON: ") + len("invalid JSON: ")
        assert b[:k] == a[:k], (a, b)
    else:
        assert a == b, (a, b)


@pytest.mark.parametrize("pattern,seed,windows", [(0, 1, 1), (1, 7, 2), (2, 123456789012, 3)])
def test_roundtrip_reference_serialized(ref, pattern, seed, windows):
    text = ref.serialize_built_trace(pattern, 12.0, 40.0, seed, windows)
    tr = _same(ref, text)
    assert len(tr) > 100


def test_large_trace_multithreaded(ref):
    """> 1 MB: parsed in several chunks on several threads."""
    text = ref.serialize_built_trace(1, 50.0, 600.0, 5, 2)
    assert len(text) > (3 << 20)
    _same(ref, text)


HDR = b'{"trace_version":1,"pattern":"uniform","seed":3,"rate":2.5,"duration":30.0}\n'


def _rec(i, t, lang="python", cls="completion", pr=256, out=50, **extra):
    d = {"request_id": i, "arrival_time_s": t, "language": lang, "task_class": cls, "prompt_tokens": pr,
         "output_tokens": out}
    d.update(extra)
    return json.dumps(d).encode() + b"\n"


def test_format_variations(ref):
    body = (b"\n\n" + HDR + b"\n" + _rec(0, 0.5) + b"\r\n"[1:] +
            b'{"output_tokens":600,"prompt_tokens":512,"task_class":"reasoning","language":"go",'
            b'"arrival_time_s":1,"request_id":1,"x":{"a":[1,2,{"b":null}]},"y":[true,false]}\n' +
            b'{"request_id":2,"arrival_time_s":1.5e0,"language":"c","task_class":"completion",'
            b'"prompt_tokens":256.9,"output_tokens":50,"note":"\\u00e9\\ud83d\\ude00\\n"}\r\n' +
            b'{"request_id":3,"request_id":4,"arrival_time_s":2,"language":"rust","task_class":"completion",'
            b'"prompt_tokens":true,"output_tokens":50}\n' +
            _rec(5, 2.0, lang="javascript") + _rec(6, 1e20, lang="csharp", cls="reasoning"))
    _same(ref, body)
    _same(ref, HDR.rstrip(b"\n"))  # header only, no newline
    _same(ref, HDR.replace(b"}", b',"windows":4}'))


@pytest.mark.parametrize("text", [
    b"",
    b"\n\n",
    b'{"pattern":"uniform"}\n',
    b'[1,2]\n',
    b'{"trace_version":2,"pattern":"uniform","seed":1,"rate":1,"duration":1}\n',
    b'{"trace_version":1,"pattern":"bursty","seed":1,"rate":1,"duration":1}\n',
    b'{"trace_version":1,"pattern":"uniform","seed":"1","rate":1,"duration":1}\n',
    b'{"trace_version":1,"pattern":"uniform","seed":1,"duration":1}\n',
    b'{"trace_version":1,"pattern":"uniform","seed":1,"rate":1,"duration":1,"windows":"2"}\n',
    HDR + _rec(0, 1.0, lang="fortran"),
    HDR + _rec(0, 1.0, cls="chat"),
    HDR + b'{"arrival_time_s":1,"language":"go","task_class":"completion","prompt_tokens":1,"output_tokens":1}\n',
    HDR + b'{"request_id":0,"arrival_time_s":"1","language":"go","task_class":"completion",'
          b'"prompt_tokens":1,"output_tokens":1}\n',
    HDR + b'{"request_id":0,"arrival_time_s":1,"language":5,"task_class":"completion",'
          b'"prompt_tokens":1,"output_tokens":1}\n',
    HDR + b'{"request_id":true,"arrival_time_s":1,"language":"go","task_class":"completion",'
          b'"prompt_tokens":1,"output_tokens":1}\n',
    HDR + b'{"request_id":0,"arrival_time_s":null,"language":"go","task_class":"completion",'
          b'"prompt_tokens":1,"output_tokens":1}\n',
    HDR + b'[1,2]\n',
    HDR + b'"just a string"\n',
    HDR + _rec(0, -1.0),
    HDR + _rec(0, 1.0, pr=0),
    HDR + _rec(0, 1.0, out=-5),
    HDR + _rec(0, 2.0) + _rec(1, 1.0),
    HDR + _rec(0, 2.0) + b"\n" + _rec(1, 3.0) + _rec(2, 2.5),
])
def test_errors_match_reference(ref, text):
    _err(ref, text)


@pytest.mark.parametrize("text", [
    b"{\n",
    b'{"trace_version":1,\n',
    HDR + b'{"request_id":0,}\n',
    HDR + b'{"request_id":01}\n',
    HDR + b"   \n",
    HDR + b'{"a":1} x\n',
    HDR + b"\r\n\r\n",
])
def test_syntax_errors_same_prefix(ref, text):
    _err(ref, text, prefix_only=True)


def test_number_overflow_matches_reference_text(ref):
    """Overflowing literals are a parse error in nlohmann (out_of_range.406);
    found by the fuzz test — the full message matches."""
    _err(ref, HDR + _rec(0, 1.0).replace(b'"arrival_time_s": 1.0', b'"arrival_time_s": 4.2e999'))
    _err(ref, HDR.replace(b'"rate":2.5', b'"rate":-1e400'))


def test_out_of_order_across_chunks(ref):
    """The arrival-order check spans the per-thread chunk boundaries."""
    lines = [HDR]
    t = 0.0
    for i in range(60000):
        t += 0.01
        lines.append(_rec(i, round(t, 2)))
    lines[40000] = _rec(39999, 0.5)  # goes backwards deep inside the file
    _err(ref, b"".join(lines))


def test_load_trace_file(ref, tmp_path):
    text = ref.serialize_built_trace(0, 5.0, 30.0, 2, 1)
    p = tmp_path / "t.jsonl"
    p.write_bytes(text)
    tr, hdr, _ = api.load_trace(str(p), api.ModelCatalog.build_default())
    tr2, _, _ = _ours(text)
    assert np.array_equal(tr.arrival_time_s, tr2.arrival_time_s) and hdr.seed == 2
    with pytest.raises(api.SimError) as e:
        api.load_trace(str(tmp_path / "missing.jsonl"), api.ModelCatalog.build_default())
    assert str(e.value) == "trace: cannot open: " + str(tmp_path / "missing.jsonl")


def test_fuzz_against_reference(ref):
    """Randomly mutated traces (dropped / duplicated / retyped fields, junk
    bytes, reordered lines, extra keys): the parsed trace or the error text
    equals the reference parser's (syntax errors: same prefix)."""
    rng = np.random.default_rng(77)
    base = ref.serialize_built_trace(2, 8.0, 20.0, 9, 1).split(b"\n")
    mutations = 0
    for case in range(300):
        lines = list(base)
        for _ in range(int(rng.integers(1, 4))):
            i = int(rng.integers(0, len(lines)))
            op = int(rng.integers(0, 9))
            ln = lines[i]
            if op == 0:
                lines[i] = ln.replace(b'"prompt_tokens"', b'"prompt_token"', 1)
            elif op == 1:
                lines[i] = ln.replace(b'"python"', b'"cobol"', 1)
            elif op == 2 and len(ln) > 3:
                j = int(rng.integers(1, len(ln)))
                lines[i] = ln[:j] + bytes([int(rng.integers(32, 127))]) + ln[j + 1:]
            elif op == 3 and len(ln) > 3:
                lines[i] = ln[: int(rng.integers(1, len(ln)))]
            elif op == 4 and i + 1 < len(lines):
                lines[i], lines[i + 1] = lines[i + 1], lines[i]
            elif op == 5:
                lines[i] = ln.replace(b"}", b',"extra":{"a":[1,2.5e3,"x"]}}', 1)
            elif op == 6:
                lines[i] = ln.replace(b'"output_tokens":', b'"output_tokens":"', 1)
            elif op == 7:
                lines.insert(i, b"")
            else:
                lines[i] = ln.replace(b'"arrival_time_s":', b'"arrival_time_s":-', 1)
            mutations += 1
        text = b"\n".join(lines)
        try:
            want = ref.parse_trace(text)
            err = None
        except Exception as e:  # noqa: BLE001
            want, err = None, str(e)
        if err is None:
            tr, hdr, rid = _ours(text)
            assert np.array_equal(tr.arrival_time_s.view(np.uint64), want["arrival"].view(np.uint64)), case
            assert np.array_equal(rid, want["request_id"]) and np.array_equal(tr.output_tokens, want["output"]), case
        else:
            with pytest.raises(api.SimError) as e_ours:
                _ours(text)
            got = str(e_ours.value)
            if "invalid JSON: " in err:
                k = err.index("invalid JSON: ") + len("invalid JSON: ")
                assert got[:k] == err[:k], (case, err, got)
            else:
                assert got == err, (case, err, got)
    assert mutations > 300


def test_bom_utf8_and_deep_nesting(ref):
    """Advisor round 1: a UTF-8 BOM at the start of a line is skipped (nlohmann
    skip_bom), a partial BOM is an error, ill-formed UTF-8 inside a string is
    an error (parse_error.101), well-formed multi-byte UTF-8 passes, and an
    ignored field may nest deeper than 512 (nlohmann's parser has no limit)."""
    bom = b"\xef\xbb\xbf"
    _same(ref, bom + HDR + _rec(0, 0.5) + _rec(1, 1.0))
    _same(ref, HDR + bom + _rec(0, 0.5) + _rec(1, 1.0))
    _err(ref, b"\xef\xbb" + HDR + _rec(0, 0.5), prefix_only=True)
    good = ['"\xc3\xa9"', '"\xe2\x82\xac"', '"\xf0\x9f\x98\x80"', '"\xed\x9f\xbf"', '"\xf4\x8f\xbf\xbf"']
    for g in good:
        line = _rec(0, 0.5)[:-2] + b',"note":' + g.encode("latin-1") + b"}\n"
        _same(ref, HDR + line)
    bad = [b'"\x80"', b'"\xc0\xaf"', b'"\xc3"', b'"\xe0\x80\x80"', b'"\xed\xa0\x80"', b'"\xf0\x80\x80\x80"',
           b'"\xf4\x90\x80\x80"', b'"\xf5\x80\x80\x80"', b'"\xe2\x82"']
    for b_ in bad:
        line = _rec(0, 0.5)[:-2] + b',"note":' + b_ + b"}\n"
        _err(ref, HDR + line, prefix_only=True)
    deep = b"[" * 3000 + b"]" * 3000
    _same(ref, HDR + _rec(0, 0.5)[:-2] + b',"deep":' + deep + b"}\n")
    deep_obj = b'{"a":' * 1500 + b"1" + b"}" * 1500
    _same(ref, HDR + _rec(0, 0.5)[:-2] + b',"deep":' + deep_obj + b"}\n")
    _err(ref, HDR + _rec(0, 0.5)[:-2] + b',"deep":' + b"[" * 700 + b"]" * 699 + b"}\n", prefix_only=True)
