"""The einsum mirror (paper_2503_04771_b200.einsum) against the reference:
parse / derive_maps results and error messages on 629 specs recorded from
bridgegen (tests/golden/parse_golden.json), the printed-module golden texts,
and the checks of bridgegen's test_einsum.py (re-stated on this API)."""

import pytest

import _golden as G
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200.einsum import EinsumError, parse_einsum


@pytest.mark.parametrize("row", G.parse_cases(), ids=range(len(G.parse_cases())))
def test_parse_matches_reference(row):
    t = row["text"]
    if row["ok"]:
        s = parse_einsum(t)
        maps, its = E.derive_maps(s)
        assert [list(x) for x in s.inputs] == row["inputs"]
        assert list(s.output) == row["output"]
        assert list(s.axes) == row["axes"]
        assert [[m.n_axes, list(m.targets)] for m in maps] == row["maps"]
        assert its == row["iterators"]
    else:
        with pytest.raises(EinsumError) as ei:
            parse_einsum(t)
        assert str(ei.value) == row["error"]


@pytest.mark.parametrize("key", sorted(G.printed_cases()))
def test_printed_module_matches_reference(key):
    text, elem = key.split("|")
    got = E.print_module(E.build_einsum_function(None, parse_einsum(text), elem=elem))
    assert got == G.printed_cases()[key]


class TestReferenceEinsumSuite:
    """test_einsum.py:16-160 restated against this package."""

    def test_matmul(self):
        spec = parse_einsum("(i,k),(k,j)->(i,j)")
        assert spec.inputs == (("i", "k"), ("k", "j"))
        assert spec.output == ("i", "j")
        assert spec.axes == ("i", "j", "k")

    def test_errors(self):
        with pytest.raises(EinsumError, match="does not appear in any input"):
            parse_einsum("(i,j)->(k)")
        with pytest.raises(EinsumError, match="repeated index"):
            parse_einsum("(i,i)->(i)")
        for bad in ("i,k->i", "(i,k)(k,j)->(i,j)", "(i,k)->", "->(i)", "ij,jk->ik"):
            with pytest.raises(EinsumError):
                parse_einsum(bad)

    def test_body_structure(self):
        mod = E.build_einsum_function(None, parse_einsum("(i,k),(k,j)->(i,j)"))
        op = mod.lookup_symbol("einsum").ops[0]
        assert op.body == ("arith.mulf", "arith.addf", "linalg.yield")
        assert len(op.attributes["indexing_maps"]) == 3
        mod = E.build_einsum_function(None, parse_einsum("(i)->(i)"))
        assert mod.lookup_symbol("einsum").ops[0].body == ("linalg.yield",)
        mod = E.build_einsum_function(None, parse_einsum("(i,j),(j,k),(k,l)->(i,l)"))
        assert mod.lookup_symbol("einsum").ops[0].body == (
            "arith.mulf", "arith.mulf", "arith.addf", "linalg.yield")

    def _ctx(self, types):
        return E.FunctionBuilder(E.Module(), "f", types)

    def test_rank_mismatch(self):
        ctx = self._ctx([E.TensorType(E.F32, 1)] * 3)
        with pytest.raises(EinsumError, match="rank"):
            E.build_generic(ctx, None, parse_einsum("(i,k),(k,j)->(i,j)"), list(ctx.arguments))

    def test_mixed_element_types_rejected(self):
        ctx = self._ctx([E.TensorType(E.F32, 1), E.TensorType(E.F64, 1), E.TensorType(E.F32, 1)])
        with pytest.raises(EinsumError, match="element type"):
            E.build_generic(ctx, None, parse_einsum("(i),(i)->(i)"), list(ctx.arguments))

    def test_operand_count(self):
        ctx = self._ctx([E.TensorType(E.F32, 2)] * 2)
        with pytest.raises(EinsumError, match="expected 2 input"):
            E.build_generic(ctx, None, parse_einsum("(i,k),(k,j)->(i,j)"), list(ctx.arguments))

    def test_bf16_module_prints(self):
        text = E.print_module(E.build_einsum_function(None, parse_einsum("(i,k),(k,j)->(i,j)"),
                                                      elem=E.BF16))
        assert "tensor<?x?xbf16>" in text and "arith.mulf %1, %2 : bf16" in text


def test_schedule_attribute_roundtrip():
    from paper_2503_04771_b200.schedule import Schedule, as_schedule_dict
    s = Schedule.parse("tile_n=512, cta_group=2")
    assert s == Schedule(tile_n=512, cta_group=2) and str(s) == "tile_n=512,cta_group=2"
    assert as_schedule_dict("raster=-8") == {"raster": -8}
    with pytest.raises(ValueError, match="unknown schedule parameter"):
        Schedule.parse("tiles=3")
    mod = E.build_einsum_function(None, parse_einsum("(i,k),(k,j)->(i,j)"), elem=E.BF16,
                                  schedule="tile_n=256,cta_group=1")
    op = mod.lookup_symbol("einsum").ops[0]
    assert op.attributes["bgx.schedule"] == "tile_n=256,cta_group=1"
    assert 'bgx.schedule = "tile_n=256,cta_group=1"' in E.print_module(mod)
    # without a schedule the printed text stays the reference's
    plain = E.print_module(E.build_einsum_function(None, parse_einsum("(i,k),(k,j)->(i,j)")))
    assert plain == G.printed_cases()["(i,k),(k,j)->(i,j)|f32"]
