"""The feasibility sweep API's host side (feasibility.hpp), on CPU, against
the reference's own feasibility.cpp (oracle/_ref/libcolorvibe_ref_codec.so):
config JSON text and hash byte for byte, its parser's acceptance and
messages, and the reference's test_feasibility.cpp host cases."""
import pytest

CONFIGS = [
    '{"version": 1}',
    '{"version": 1, "delta_basis": "frame_diff"}',
    '{"version": 1, "delta_mode": "continuous", "workers": 3}',
    '{"version": 1, "grid": {"radius": {"min": 1, "max": 5, "step": 2}, '
    '"angle_deg": {"min": 0, "max": 90, "step": 45}}}',
    '{"version": 1, "grid": {"radius": {"min": 1, "max": 2, "step": 1}, '
    '"angle_deg": {"min": 0, "max": 350, "step": 10}}, "half_sweep": true}',
    '{"version": 1, "grid": {"radii": [0.5, 1.25, 7], "angles_rad": [0, 0.1, 3.14159]}}',
    '{"version": 1, "colors": [{"name": "a\\"b", "rgb": [1, 2, 3]}, {"name": "c", "rgb": [255, 0, 7]}], '
    '"patterns": ["111", "001"], "v_th": [7.5, 1e-3, 254.99], "r_novib": [1, 0.015625], '
    '"white_point": [0.9642, 1.0, 0.8251]}',
]

BAD = [
    "{}", '{"version": 2}', "not json", '{"version": 1, "patterns": ["000"]}',
    '{"version": 1, "delta_basis": "nope"}', '{"version": 1.0}', "[1]",
    '{"version": 1, "colors": []}', '{"version": 1, "colors": [{"name": "x", "rgb": [1, 2]}]}',
    '{"version": 1, "colors": [{"name": "x", "rgb": [1, 2, 3]}, {"name": "x", "rgb": [1, 2, 3]}]}',
    '{"version": 1, "v_th": [0]}', '{"version": 1, "r_novib": [1.5]}', '{"version": 1, "workers": -1}',
    '{"version": 1, "white_point": [1, 2]}', '{"version": 1, "grid": {"radii": [2, 1], "angles_rad": [0]}}',
    '{"version": 1, "grid": {"radius": {"min": 1}}}', '{"version": 1, "v_th": "x"}',
    '{"version": 1, "half_sweep": 1}',
]


@pytest.mark.parametrize("text", CONFIGS)
def test_config_text_and_hash_match_reference(cv, ref_codec, text):
    ref_text, ref_hash = ref_codec.config_roundtrip(text)
    cfg = cv.config_from_json(text)
    assert cv.config_to_json(cfg) == ref_text
    assert cv.config_hash(cfg) == ref_hash
    assert cv.config_to_json(cv.config_from_json(ref_text)) == ref_text  # idempotent


@pytest.mark.parametrize("text", BAD)
def test_bad_configs_rejected_like_reference(cv, ref_codec, text):
    with pytest.raises(ValueError) as ref:
        ref_codec.config_roundtrip(text)
    with pytest.raises(ValueError) as ours:
        cv.config_from_json(text)
    msg_ref, msg_ours = str(ref.value), str(ours.value)
    # nlohmann's own exception texts (parse errors, type errors) are not
    # restated word for word; everything the reference words itself is
    if "json.exception" in msg_ref:
        assert msg_ours.split(":")[0] == msg_ref.split(":")[0]
    else:
        assert msg_ours == msg_ref


def test_default_config_shape(cv):  # test_feasibility.cpp:34-53
    cfg = cv.SearchConfig.defaults()
    assert len(cfg.colors) == 9 and len(cfg.patterns) == 7
    assert cfg.v_th_values == [50.0, 100.0, 150.0, 200.0]
    assert cfg.r_novib_values == [0.5, 0.25, 0.125]
    assert len(cfg.grid.radii) == 6 and len(cfg.grid.angles) == 30
    assert cfg.combo_count() == 756
    cfg.validate()
    assert cfg.colors[0].name == "Black" and cfg.colors[0].rgb == cv.SrgbColor(100, 100, 100)
    assert cfg.colors[-1].name == "Magenta" and cfg.colors[-1].rgb == cv.SrgbColor(240, 100, 240)
    bench = cv.SearchConfig.benchmark_defaults()
    assert bench.grid.candidate_count() == 36000 and bench.combo_count() == 756
    assert cfg.delta_basis == cv.DeltaBasis.TARGET_SWING


def test_degenerate_configs_rejected(cv):  # test_feasibility.cpp:172-190
    cfg = cv.SearchConfig.defaults()
    cfg.colors = []
    with pytest.raises(ValueError):
        cfg.validate()
    cfg = cv.SearchConfig.defaults()
    cfg.colors = cfg.colors + [cfg.colors[0]]
    with pytest.raises(ValueError, match="duplicate color name Black"):
        cfg.validate()
    cfg = cv.SearchConfig.defaults()
    g = cfg.grid
    g.radii = []
    cfg.grid = g
    with pytest.raises(ValueError, match="degenerate grid"):
        cfg.validate()
    cfg = cv.SearchConfig.defaults()
    cfg.v_th_values = [0.0]
    with pytest.raises(ValueError, match="v_th values must be positive"):
        cfg.validate()


def test_export_names(cv):  # test_feasibility.cpp:166-170
    assert cv.matrix_filename("csv", True) == "matrix_aggregated.csv"
    assert cv.matrix_filename("json", False) == "matrix_full.json"
    with pytest.raises(ValueError, match="unsupported format: xml"):
        cv.matrix_filename("xml", True)
