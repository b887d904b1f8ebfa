// bindings.cpp -- Python module `_core`, mirroring the reference binding
// (proj/bindings/module.cpp:18-131: the types and the search functions) plus
// a NumPy batch interface and device-resident plans for pipelines/benchmarks.
// batch_search releases the GIL like the reference (module.cpp:121-131).
#include <pybind11/numpy.h>
#include <pybind11/operators.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <numbers>
#include <sstream>
#include <stdexcept>

#include "../../include/cvg.h"
#include "colorvibe/bench.hpp"
#include "colorvibe/codec.hpp"
#include "colorvibe/feasibility.hpp"
#include "colorvibe/search.hpp"

namespace py = pybind11;
using namespace colorvibe;

namespace {

void check(int status) {
    if (status == CVG_OK) return;
    const std::string msg = cvg_last_error();
    if (status == CVG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct Context;

// Owns a cvg_result; NumPy arrays view its buffers (zero copy).  It keeps
// the context alive: the buffers are blocks of the context's pinned pool.
struct ResultHolder {
    cvg_result r{};
    std::shared_ptr<Context> owner;
    ~ResultHolder() { cvg_result_free(&r); }
};

int out_mode(const std::string& s) {
    if (s == "pairs") return CVG_OUT_PAIRS;
    if (s == "counts") return CVG_OUT_COUNTS;
    if (s == "first") return CVG_OUT_FIRST;
    if (s == "best") return CVG_OUT_BEST;
    throw std::invalid_argument("output must be 'pairs', 'counts', 'first' or 'best'");
}

int path_mode(const std::string& s) {
    if (s == "fast") return CVG_PATH_FAST;
    if (s == "exact") return CVG_PATH_EXACT;
    if (s == "audit") return CVG_PATH_AUDIT;
    if (s == "pruned") return CVG_PATH_PRUNED;
    if (s == "memo") return CVG_PATH_MEMO;
    throw std::invalid_argument("path must be 'fast', 'exact', 'audit', 'pruned' or 'memo'");
}

using I32 = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;
using F64 = py::array_t<double, py::array::c_style | py::array::forcecast>;

// Arrays kept alive for the duration of a descriptor's use.
struct Desc {
    I32 rgb, bits;
    F64 vth, rn, radii, angles;
    std::vector<double> wp;
    cvg_search_desc d{};

    Desc(I32 rgb_, I32 bits_, F64 vth_, F64 rn_, F64 radii_, F64 angles_, int mode, int basis, py::object white,
         const std::string& output, const std::string& path)
        : rgb(std::move(rgb_)), bits(std::move(bits_)), vth(std::move(vth_)), rn(std::move(rn_)),
          radii(std::move(radii_)), angles(std::move(angles_)) {
        const py::ssize_t n = bits.size();
        if (rgb.size() != 3 * n || vth.size() != n || rn.size() != n) {
            throw std::invalid_argument("targets must be (n, 3); patterns, v_th, r_novib must be (n,)");
        }
        d.n_searches = static_cast<int32_t>(n);
        d.target_rgb = rgb.data();
        d.pattern_bits = bits.data();
        d.v_th = vth.data();
        d.r_novib = rn.data();
        d.n_radii = static_cast<int32_t>(radii.size());
        d.radii = radii.data();
        d.n_angles = static_cast<int32_t>(angles.size());
        d.angles = angles.data();
        d.delta_mode = mode;
        d.delta_basis = basis;
        if (!white.is_none()) {
            wp = white.cast<std::vector<double>>();
            if (wp.size() != 3) throw std::invalid_argument("white_point must have 3 entries");
            d.white_point = wp.data();
        }
        d.output = out_mode(output);
        d.path = path_mode(path);
    }
};

py::dict result_dict(std::shared_ptr<ResultHolder> h, int output) {
    py::object base = py::cast(h);
    const cvg_result& r = h->r;
    py::dict out;
    const py::ssize_t n = r.n_searches;
    out["counts"] = py::array_t<uint64_t>({n}, {sizeof(uint64_t)}, r.counts, base);  // pinned, zero-copy
    out["n_pairs"] = r.n_pairs;
    if (output == CVG_OUT_PAIRS) {
        out["offsets"] = py::array_t<uint64_t>({n + 1}, {sizeof(uint64_t)}, r.offsets, base);
        const py::ssize_t np_ = static_cast<py::ssize_t>(r.n_pairs);
        if (np_) {
            out["idx"] = py::array_t<uint32_t>({np_}, {sizeof(uint32_t)}, r.idx, base);
            out["codes"] = py::array_t<uint8_t>({np_, py::ssize_t(6)}, {py::ssize_t(6), py::ssize_t(1)}, r.codes, base);
        } else {
            out["idx"] = py::array_t<uint32_t>(0);
            out["codes"] = py::array_t<uint8_t>(std::vector<py::ssize_t>{0, 6});
        }
    } else if (output == CVG_OUT_FIRST || output == CVG_OUT_BEST) {
        if (n) {
            out["first_idx"] = py::array_t<uint32_t>({n}, {sizeof(uint32_t)}, r.first_idx, base);
            out["first_codes"] = py::array_t<uint8_t>({n, py::ssize_t(6)}, {py::ssize_t(6), py::ssize_t(1)}, r.first_codes, base);
        } else {
            out["first_idx"] = py::array_t<uint32_t>(0);
            out["first_codes"] = py::array_t<uint8_t>(std::vector<py::ssize_t>{0, 6});
        }
    }
    py::dict stats;
    stats["candidates"] = r.n_candidates;
    stats["band_repairs"] = r.n_band_repairs;
    stats["code_repairs"] = r.n_code_repairs;
    stats["audit_violations"] = r.n_audit_violations;
    stats["class_mismatch"] = r.n_class_mismatch;
    stats["audit_max_ratio"] = r.audit_max_ratio;
    stats["kernel_ms"] = r.kernel_ms;
    stats["h2d_bytes"] = r.h2d_bytes;
    stats["d2h_bytes"] = r.d2h_bytes;
    stats["prep_ms"] = r.prep_ms;
    stats["h2d_ms"] = r.h2d_ms;
    stats["device_ms"] = r.device_ms;
    stats["d2h_ms"] = r.d2h_ms;
    stats["total_ms"] = r.total_ms;
    out["stats"] = stats;
    return out;
}

struct Context {
    cvg_ctx* ctx = nullptr;
    explicit Context(int device) { check(cvg_create(device, &ctx)); }
    ~Context() { cvg_destroy(ctx); }
};

struct Plan {
    std::shared_ptr<Context> ctx;
    std::unique_ptr<Desc> desc;
    cvg_plan* plan = nullptr;
    int output = 0;
    ~Plan() { cvg_plan_destroy(plan); }
};

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200 color-vibration pair search (drop-in for colorvibe._core search API)";

    // ---- reference types (module.cpp:18-104) ----
    py::class_<SrgbColor>(m, "SrgbColor")
        .def(py::init<int, int, int>(), py::arg("r"), py::arg("g"), py::arg("b"))
        .def_readwrite("r", &SrgbColor::r)
        .def_readwrite("g", &SrgbColor::g)
        .def_readwrite("b", &SrgbColor::b)
        .def(py::self == py::self)
        .def("__repr__", [](const SrgbColor& c) {
            std::ostringstream s;
            s << "SrgbColor(" << c.r << ", " << c.g << ", " << c.b << ")";
            return s.str();
        });

    py::class_<LabColor>(m, "LabColor")
        .def(py::init<double, double, double>(), py::arg("l"), py::arg("a"), py::arg("b"))
        .def_readwrite("l", &LabColor::l)
        .def_readwrite("a", &LabColor::a)
        .def_readwrite("b", &LabColor::b)
        .def("__repr__", [](const LabColor& c) {
            std::ostringstream s;
            s << "LabColor(" << c.l << ", " << c.a << ", " << c.b << ")";
            return s.str();
        });

    py::class_<WhitePoint>(m, "WhitePoint")
        .def(py::init<double, double, double>(), py::arg("x"), py::arg("y"), py::arg("z"))
        .def_readwrite("x", &WhitePoint::x)
        .def_readwrite("y", &WhitePoint::y)
        .def_readwrite("z", &WhitePoint::z);

    py::class_<BitPattern>(m, "BitPattern")
        .def(py::init([](const std::string& s) { return BitPattern::parse(s); }), py::arg("bits"))
        .def_static("parse", &BitPattern::parse)
        .def_readwrite("r", &BitPattern::r)
        .def_readwrite("g", &BitPattern::g)
        .def_readwrite("b", &BitPattern::b)
        .def("any", &BitPattern::any)
        .def(py::self == py::self)
        .def("__str__", &BitPattern::str)
        .def("__repr__", [](const BitPattern& p) { return "BitPattern(\"" + p.str() + "\")"; });

    py::class_<Thresholds>(m, "Thresholds")
        .def(py::init<double, double>(), py::arg("v_th"), py::arg("r_novib"))
        .def_readwrite("v_th", &Thresholds::v_th)
        .def_readwrite("r_novib", &Thresholds::r_novib)
        .def("low_band", &Thresholds::low_band)
        .def("validate", &Thresholds::validate);

    py::class_<VibrationGrid>(m, "VibrationGrid")
        .def(py::init<>())
        .def_static("uniform", &VibrationGrid::uniform, py::arg("radius_min"), py::arg("radius_max"),
                    py::arg("radius_step"), py::arg("angle_min_deg"), py::arg("angle_max_deg"),
                    py::arg("angle_step_deg"))
        .def_static("standard", &VibrationGrid::standard)
        .def_readwrite("radii", &VibrationGrid::radii)
        .def_readwrite("angles", &VibrationGrid::angles)
        .def("candidate_count", &VibrationGrid::candidate_count)
        .def("validate", &VibrationGrid::validate);

    py::class_<ChannelDeltas>(m, "ChannelDeltas")
        .def(py::init<double, double, double>(), py::arg("dr") = 0.0, py::arg("dg") = 0.0, py::arg("db") = 0.0)
        .def_readonly("dr", &ChannelDeltas::dr)
        .def_readonly("dg", &ChannelDeltas::dg)
        .def_readonly("db", &ChannelDeltas::db)
        .def(py::self == py::self)
        .def("__repr__", [](const ChannelDeltas& d) {
            std::ostringstream s;
            s << "ChannelDeltas(" << d.dr << ", " << d.dg << ", " << d.db << ")";
            return s.str();
        });

    py::class_<ColorPair>(m, "ColorPair")
        .def(py::init([](SrgbColor target, SrgbColor plus, SrgbColor minus, double radius, double angle,
                         ChannelDeltas deltas) { return ColorPair{target, plus, minus, radius, angle, deltas}; }),
             py::arg("target") = SrgbColor{}, py::arg("plus") = SrgbColor{}, py::arg("minus") = SrgbColor{},
             py::arg("radius") = 0.0, py::arg("angle") = 0.0, py::arg("deltas") = ChannelDeltas{})
        .def_readonly("target", &ColorPair::target)
        .def_readonly("plus", &ColorPair::plus)
        .def_readonly("minus", &ColorPair::minus)
        .def_readonly("radius", &ColorPair::radius)
        .def_readonly("angle", &ColorPair::angle)
        .def_readonly("deltas", &ColorPair::deltas)
        .def(py::self == py::self)
        .def_property_readonly("angle_deg", [](const ColorPair& p) { return p.angle * 180.0 / std::numbers::pi; })
        .def("__repr__", [](const ColorPair& p) {
            std::ostringstream s;
            s << "ColorPair(r=" << p.radius << ", angle=" << p.angle << ", plus=(" << p.plus.r << "," << p.plus.g
              << "," << p.plus.b << "), minus=(" << p.minus.r << "," << p.minus.g << "," << p.minus.b << "))";
            return s.str();
        });

    py::enum_<DeltaMode>(m, "DeltaMode")
        .value("QUANTIZED", DeltaMode::Quantized)
        .value("CONTINUOUS", DeltaMode::Continuous);
    py::enum_<DeltaBasis>(m, "DeltaBasis")
        .value("TARGET_SWING", DeltaBasis::TargetSwing)
        .value("FRAME_DIFF", DeltaBasis::FrameDiff);

    py::class_<SearchOptions>(m, "SearchOptions")
        .def(py::init<>())
        .def_readwrite("delta_mode", &SearchOptions::delta_mode)
        .def_readwrite("delta_basis", &SearchOptions::delta_basis)
        .def_readwrite("workers", &SearchOptions::workers)
        .def_readwrite("white_point", &SearchOptions::white_point);

    py::class_<SearchSpec>(m, "SearchSpec")
        .def(py::init<SrgbColor, BitPattern, Thresholds>(), py::arg("target"), py::arg("pattern"),
             py::arg("thresholds"))
        .def_readwrite("target", &SearchSpec::target)
        .def_readwrite("pattern", &SearchSpec::pattern)
        .def_readwrite("thresholds", &SearchSpec::thresholds);

    // ---- reference functions (module.cpp:106-139) ----
    m.def("d65_white", &d65_white, py::return_value_policy::copy);
    m.def("srgb_to_lab", [](const SrgbColor& c) { return srgb_to_lab(c); }, py::arg("color"));
    m.def("lab_to_srgb", [](const LabColor& c) { return lab_to_srgb(c); }, py::arg("color"),
          "Returns None when the color falls outside the sRGB gamut");
    m.def("lab_to_srgb_clipped", [](const LabColor& c) { return lab_to_srgb_clipped(c); }, py::arg("color"),
          "Clamps out-of-gamut channels before quantizing");
    m.def("in_gamut", [](const LabColor& c) { return in_gamut(c); }, py::arg("color"));
    m.def("srgb_to_linear", &srgb_to_linear, py::arg("code"));
    m.def("displaced_pair", &displaced_pair, py::arg("target"), py::arg("radius"), py::arg("angle"));
    m.def(
        "serial_search",
        [](const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern, const Thresholds& th,
           int workers) {
            SearchOptions opts;
            opts.workers = workers;
            return serial_search(target, grid, pattern, th, opts);
        },
        py::arg("target"), py::arg("grid"), py::arg("pattern"), py::arg("thresholds"), py::arg("workers") = 0,
        py::call_guard<py::gil_scoped_release>());
    m.def(
        "batch_search",
        [](const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern, const Thresholds& th,
           int workers) {
            SearchOptions opts;
            opts.workers = workers;
            return batch_search(target, grid, pattern, th, opts);
        },
        py::arg("target"), py::arg("grid"), py::arg("pattern"), py::arg("thresholds"), py::arg("workers") = 0,
        py::call_guard<py::gil_scoped_release>());
    // Lazy result (B200 extension): the packed records stay in pinned host
    // memory; ColorPair objects are built on access.  Compares equal to the
    // list batch_search returns.
    py::class_<PairView>(m, "PairView")
        .def("__len__", &PairView::size)
        .def("__getitem__", [](const PairView& v, py::ssize_t i) {
            const py::ssize_t n = static_cast<py::ssize_t>(v.size());
            if (i < 0) i += n;
            if (i < 0 || i >= n) throw py::index_error("PairView index out of range");
            return v.at(static_cast<size_t>(i));
        })
        .def("__getitem__", [](const PairView& v, const py::slice& sl) {
            size_t start = 0, stop = 0, step = 0, len = 0;
            if (!sl.compute(v.size(), &start, &stop, &step, &len)) throw py::error_already_set();
            std::vector<ColorPair> out;
            out.reserve(len);
            for (size_t j = 0; j < len; ++j) out.push_back(v.at(start + j * step));
            return out;
        })
        .def("__iter__", [](py::object self) {
            return py::iter(py::module_::import("builtins").attr("map")(self.attr("__getitem__"),
                                                                        py::module_::import("builtins").attr("range")(
                                                                            py::len(self))));
        })
        .def("__eq__", [](const PairView& v, py::object other) {
            if (py::isinstance<PairView>(other)) {
                const PairView& o = other.cast<const PairView&>();
                if (o.size() != v.size()) return false;
                for (size_t i = 0; i < v.size(); ++i) if (!(v.at(i) == o.at(i))) return false;
                return true;
            }
            if (!py::isinstance<py::sequence>(other)) return false;
            py::sequence seq = other;
            if (static_cast<size_t>(py::len(seq)) != v.size()) return false;
            for (size_t i = 0; i < v.size(); ++i) {
                py::object x = seq[i];
                if (!py::isinstance<ColorPair>(x) || !(x.cast<const ColorPair&>() == v.at(i))) return false;
            }
            return true;
        })
        .def("__bool__", [](const PairView& v) { return !v.empty(); })
        .def("__repr__", [](const PairView& v) { return "PairView(" + std::to_string(v.size()) + " pairs)"; })
        .def("to_list", &PairView::to_vector, py::call_guard<py::gil_scoped_release>())
        .def_property_readonly("idx", [](py::object self) {
            const PairView& v = self.cast<const PairView&>();
            const py::ssize_t n = static_cast<py::ssize_t>(v.size());
            if (!n) return py::array_t<uint32_t>(0);
            return py::array_t<uint32_t>({n}, {sizeof(uint32_t)}, v.idx(), self);  // zero-copy
        })
        .def_property_readonly("codes", [](py::object self) {
            const PairView& v = self.cast<const PairView&>();
            const py::ssize_t n = static_cast<py::ssize_t>(v.size());
            if (!n) return py::array_t<uint8_t>(std::vector<py::ssize_t>{0, 6});
            return py::array_t<uint8_t>({n, py::ssize_t(6)}, {py::ssize_t(6), py::ssize_t(1)}, v.codes(), self);
        });
    m.def(
        "batch_search_view",
        [](const SrgbColor& target, const VibrationGrid& grid, const BitPattern& pattern, const Thresholds& th,
           int workers, py::object options) {
            SearchOptions opts = options.is_none() ? SearchOptions{} : options.cast<SearchOptions>();
            opts.workers = workers;
            py::gil_scoped_release nogil;
            return batch_search_view(target, grid, pattern, th, opts);
        },
        py::arg("target"), py::arg("grid"), py::arg("pattern"), py::arg("thresholds"), py::arg("workers") = 0,
        py::arg("options") = py::none());
    // Options-aware forms of the C++ API (search.hpp:126-130 take SearchOptions).
    m.def("batch_search_opts", &batch_search, py::arg("target"), py::arg("grid"), py::arg("pattern"),
          py::arg("thresholds"), py::arg("options"), py::call_guard<py::gil_scoped_release>());
    m.def("serial_search_opts", &serial_search, py::arg("target"), py::arg("grid"), py::arg("pattern"),
          py::arg("thresholds"), py::arg("options"), py::call_guard<py::gil_scoped_release>());
    m.def("batch_search_many", &batch_search_many, py::arg("specs"), py::arg("grid"),
          py::arg("options") = SearchOptions{}, py::call_guard<py::gil_scoped_release>());
    m.def("batch_count_many", &batch_count_many, py::arg("specs"), py::arg("grid"),
          py::arg("options") = SearchOptions{}, py::call_guard<py::gil_scoped_release>());
    m.def("channel_deltas", &channel_deltas, py::arg("target"), py::arg("plus"), py::arg("minus"));
    m.def("frame_deltas", &frame_deltas, py::arg("plus"), py::arg("minus"));
    m.def("classify_pair", &classify_pair, py::arg("deltas"), py::arg("pattern"), py::arg("thresholds"),
          "True when every channel delta satisfies its bit's band");
    m.def("classification_margin", &classification_margin, py::arg("pair"), py::arg("thresholds"));
    m.def("select_best", &select_best, py::arg("pairs"), py::arg("thresholds"), py::return_value_policy::copy);

    // ---- low-level C-ABI access (NumPy in / NumPy out) ----
    m.def("version", [] { return std::string(cvg_version()); });
    m.def("quant_thresholds", [] {
        py::array_t<double> a(256);
        cvg_quant_thresholds(a.mutable_data());
        return a;
    });
    m.def("measure_ffma_peak", [](int device) {
        float ms = 0.f;
        const double v = cvg_measure_ffma_peak(device, &ms);
        return py::make_tuple(v, ms);
    }, py::arg("device") = 0);

    py::class_<Context, std::shared_ptr<Context>>(m, "Context")
        .def(py::init<int>(), py::arg("device") = 0)
        .def(
            "search",
            [](std::shared_ptr<Context> self, I32 rgb, I32 bits, F64 vth, F64 rn, F64 radii, F64 angles,
               const std::string& output, const std::string& path, int mode, int basis, py::object white) {
                Desc d(std::move(rgb), std::move(bits), std::move(vth), std::move(rn), std::move(radii),
                       std::move(angles), mode, basis, white, output, path);
                auto h = std::make_shared<ResultHolder>();
                h->owner = self;
                int st;
                {
                    py::gil_scoped_release nogil;
                    st = cvg_search(self->ctx, &d.d, &h->r);
                }
                check(st);
                return result_dict(h, d.d.output);
            },
            py::arg("targets"), py::arg("patterns"), py::arg("v_th"), py::arg("r_novib"), py::arg("radii"),
            py::arg("angles"), py::arg("output") = "pairs", py::arg("path") = "fast", py::arg("delta_mode") = 0,
            py::arg("delta_basis") = 0, py::arg("white_point") = py::none())
        .def(
            "plan",
            [](std::shared_ptr<Context> self, I32 rgb, I32 bits, F64 vth, F64 rn, F64 radii, F64 angles,
               const std::string& output, const std::string& path, int mode, int basis, py::object white) {
                auto p = std::make_unique<Plan>();
                p->ctx = self;
                p->desc = std::make_unique<Desc>(std::move(rgb), std::move(bits), std::move(vth), std::move(rn),
                                                 std::move(radii), std::move(angles), mode, basis, white, output, path);
                p->output = p->desc->d.output;
                check(cvg_plan_create(self->ctx, &p->desc->d, &p->plan));
                return p;
            },
            py::arg("targets"), py::arg("patterns"), py::arg("v_th"), py::arg("r_novib"), py::arg("radii"),
            py::arg("angles"), py::arg("output") = "pairs", py::arg("path") = "fast", py::arg("delta_mode") = 0,
            py::arg("delta_basis") = 0, py::arg("white_point") = py::none());

    py::class_<ResultHolder, std::shared_ptr<ResultHolder>>(m, "_Result");

    // ---- feasibility sweep (module.cpp:140-191; feasibility.hpp) ----
    py::class_<NamedColor>(m, "NamedColor")
        .def(py::init<std::string, SrgbColor>(), py::arg("name"), py::arg("rgb"))
        .def_readwrite("name", &NamedColor::name)
        .def_readwrite("rgb", &NamedColor::rgb);

    py::class_<SearchConfig>(m, "SearchConfig")
        .def(py::init(&SearchConfig::defaults))
        .def_static("defaults", &SearchConfig::defaults)
        .def_static("benchmark_defaults", &SearchConfig::benchmark_defaults)
        .def_readwrite("colors", &SearchConfig::colors)
        .def_readwrite("patterns", &SearchConfig::patterns)
        .def_readwrite("v_th_values", &SearchConfig::v_th_values)
        .def_readwrite("r_novib_values", &SearchConfig::r_novib_values)
        .def_readwrite("grid", &SearchConfig::grid)
        .def_readwrite("white_point", &SearchConfig::white_point)
        .def_readwrite("delta_mode", &SearchConfig::delta_mode)
        .def_readwrite("delta_basis", &SearchConfig::delta_basis)
        .def_readwrite("workers", &SearchConfig::workers)
        .def("validate", &SearchConfig::validate)
        .def("options", &SearchConfig::options)
        .def("combo_count", &SearchConfig::combo_count);
    m.def("config_from_json", &config_from_json, py::arg("text"));
    m.def("config_to_json", &config_to_json, py::arg("config"));
    m.def("config_hash", &config_hash, py::arg("config"));

    py::class_<FeasibilityCell>(m, "FeasibilityCell")
        .def_readonly("color_index", &FeasibilityCell::color_index)
        .def_readonly("pattern_index", &FeasibilityCell::pattern_index)
        .def_readonly("v_th_index", &FeasibilityCell::v_th_index)
        .def_readonly("r_novib_index", &FeasibilityCell::r_novib_index)
        .def_readonly("feasible", &FeasibilityCell::feasible)
        .def_readonly("pair_count", &FeasibilityCell::pair_count)
        .def_readonly("best_pair", &FeasibilityCell::best_pair);

    py::class_<FeasibilityMatrix>(m, "FeasibilityMatrix")
        .def_readonly("config", &FeasibilityMatrix::config)
        .def_readonly("cells", &FeasibilityMatrix::cells)
        .def("cell", &FeasibilityMatrix::cell, py::arg("color"), py::arg("pattern"), py::arg("v_th"),
             py::arg("r_novib"), py::return_value_policy::reference_internal);

    py::class_<AggregateMatrix>(m, "AggregateMatrix")
        .def_readonly("patterns", &AggregateMatrix::patterns)
        .def_readonly("colors", &AggregateMatrix::colors)
        .def("at", &AggregateMatrix::at, py::arg("pattern"), py::arg("color"));

    m.def("feasibility_matrix", &feasibility_matrix, py::arg("config"), py::call_guard<py::gil_scoped_release>());
    m.def("aggregate_any", &aggregate_any, py::arg("matrix"));
    m.def(
        "export_matrix",
        [](const FeasibilityMatrix& mat, const std::string& format, bool aggregated) {
            return export_matrix(mat, parse_export_format(format), aggregated);
        },
        py::arg("matrix"), py::arg("format") = "csv", py::arg("aggregated") = true);
    m.def(
        "matrix_filename",
        [](const std::string& format, bool aggregated) {
            return matrix_filename(parse_export_format(format), aggregated);
        },
        py::arg("format"), py::arg("aggregated"));

    py::class_<BenchReport>(m, "BenchReport")  // module.cpp:193-212
        .def_readonly("config_hash", &BenchReport::config_hash)
        .def_readonly("combos", &BenchReport::combos)
        .def_readonly("candidates", &BenchReport::candidates)
        .def_readonly("pairs_found", &BenchReport::pairs_found)
        .def_readonly("repetitions", &BenchReport::repetitions)
        .def_readonly("workers", &BenchReport::workers)
        .def_readonly("serial_seconds", &BenchReport::serial_seconds)
        .def_readonly("batch_seconds", &BenchReport::batch_seconds)
        .def_readonly("batch_single_seconds", &BenchReport::batch_single_seconds)
        .def_readonly("speedup", &BenchReport::speedup)
        .def_readonly("speedup_single", &BenchReport::speedup_single)
        .def_readonly("result_parity", &BenchReport::result_parity);
    m.def("run_benchmark", &run_benchmark, py::arg("config"), py::arg("repetitions") = 3,
          py::call_guard<py::gil_scoped_release>());
    m.def("bench_report_json", &bench_report_json, py::arg("report"));

    // ---- codec (module.cpp:216-296; codec.hpp, image.hpp) ----
    py::class_<Image>(m, "Image", py::buffer_protocol())
        .def_static("solid", &Image::solid, py::arg("width"), py::arg("height"), py::arg("fill"))
        .def_static("from_array", [](py::array_t<uint8_t, py::array::c_style | py::array::forcecast> a) {
            if (a.ndim() != 3 || a.shape(2) != 3) throw std::invalid_argument("expected an (height, width, 3) uint8 array");
            Image img;
            img.height = static_cast<int>(a.shape(0));
            img.width = static_cast<int>(a.shape(1));
            img.pixels.assign(a.data(), a.data() + a.size());
            return img;
        }, py::arg("array"))
        .def_readonly("width", &Image::width)
        .def_readonly("height", &Image::height)
        .def("get", &Image::get, py::arg("x"), py::arg("y"))
        .def("set", &Image::set, py::arg("x"), py::arg("y"), py::arg("color"))
        .def(py::self == py::self)
        // (height, width, 3) uint8 view of the pixels (no copy)
        .def_property_readonly("pixels", [](py::object self) {
            Image& img = self.cast<Image&>();
            return py::array_t<uint8_t>({static_cast<py::ssize_t>(img.height), static_cast<py::ssize_t>(img.width),
                                         py::ssize_t(3)},
                                        {static_cast<py::ssize_t>(3 * img.width), py::ssize_t(3), py::ssize_t(1)},
                                        img.pixels.data(), self);
        });

    py::class_<DisplayParams>(m, "DisplayParams")
        .def(py::init<>())
        .def(py::init([](double hz) {
                 DisplayParams d;
                 d.refresh_hz = hz;
                 return d;
             }),
             py::arg("refresh_hz"))
        .def_readwrite("refresh_hz", &DisplayParams::refresh_hz)
        .def_readwrite("ccff_hz", &DisplayParams::ccff_hz)
        .def("validate", &DisplayParams::validate);

    py::class_<BlockSpec>(m, "BlockSpec")
        .def(py::init<>())
        .def(py::init([](int x, int y, std::string name, SrgbColor color, BitPattern pattern) {
                 return BlockSpec{x, y, std::move(name), color, pattern};
             }),
             py::arg("x"), py::arg("y"), py::arg("color_name"), py::arg("color"), py::arg("pattern"))
        .def_readwrite("x", &BlockSpec::x)
        .def_readwrite("y", &BlockSpec::y)
        .def_readwrite("color_name", &BlockSpec::color_name)
        .def_readwrite("color", &BlockSpec::color)
        .def_readwrite("pattern", &BlockSpec::pattern);

    py::class_<BlockLayout>(m, "BlockLayout")
        .def(py::init<>())
        .def_readwrite("block_width", &BlockLayout::block_width)
        .def_readwrite("block_height", &BlockLayout::block_height)
        .def_readwrite("blocks", &BlockLayout::blocks)
        .def("validate", &BlockLayout::validate, py::arg("image_width"), py::arg("image_height"));

    py::class_<FramePair>(m, "FramePair")
        .def(py::init<>())
        .def_readwrite("frame_a", &FramePair::frame_a)
        .def_readwrite("frame_b", &FramePair::frame_b)
        .def_readwrite("layout", &FramePair::layout);

    py::enum_<BlockStatus>(m, "BlockStatus")
        .value("PATTERN", BlockStatus::Pattern)
        .value("NO_SIGNAL", BlockStatus::NoSignal)
        .value("AMBIGUOUS", BlockStatus::Ambiguous);

    py::class_<BlockResult>(m, "BlockResult")
        .def(py::init([](BlockStatus st, BitPattern p, std::array<double, 3> md) { return BlockResult{st, p, md}; }),
             py::arg("status") = BlockStatus::NoSignal, py::arg("pattern") = BitPattern{},
             py::arg("mean_deltas") = std::array<double, 3>{0.0, 0.0, 0.0})
        .def_readonly("status", &BlockResult::status)
        .def_readonly("pattern", &BlockResult::pattern)
        .def_readonly("mean_deltas", &BlockResult::mean_deltas);

    py::class_<Sidecar>(m, "Sidecar")
        .def_readonly("layout", &Sidecar::layout)
        .def_readonly("thresholds", &Sidecar::thresholds);

    m.def(
        "make_testcard",
        [](const SrgbColor& color, const BitPattern& pattern, const Thresholds& th, const VibrationGrid& grid,
           const DisplayParams& disp, int width, int height, int workers) {
            SearchOptions opts;
            opts.workers = workers;
            return make_testcard(color, pattern, th, grid, disp, width, height, opts);
        },
        py::arg("color"), py::arg("pattern"), py::arg("thresholds"), py::arg("grid"), py::arg("display"),
        py::arg("width"), py::arg("height"), py::arg("workers") = 0, py::call_guard<py::gil_scoped_release>());
    m.def(
        "embed_blocks",
        [](const Image& base, const BlockLayout& layout, const Thresholds& th, const VibrationGrid& grid,
           const DisplayParams& disp, int workers) {
            SearchOptions opts;
            opts.workers = workers;
            return embed_blocks(base, layout, th, grid, disp, opts);
        },
        py::arg("base"), py::arg("layout"), py::arg("thresholds"), py::arg("grid"), py::arg("display"),
        py::arg("workers") = 0, py::call_guard<py::gil_scoped_release>());
    m.def("embed_blocks_opts", &embed_blocks, py::arg("base"), py::arg("layout"), py::arg("thresholds"),
          py::arg("grid"), py::arg("display"), py::arg("options"), py::call_guard<py::gil_scoped_release>());
    m.def("decode_blocks", &decode_blocks, py::arg("frames"), py::arg("thresholds"),
          py::call_guard<py::gil_scoped_release>());
    m.def("layout_to_json", &layout_to_json, py::arg("layout"), py::arg("thresholds"));
    m.def("layout_from_json", &layout_from_json, py::arg("text"));
    m.def("decode_report_json", &decode_report_json, py::arg("layout"), py::arg("thresholds"), py::arg("results"));

    // ---- codec passes on device memory (C-ABI, pointers as ints) ----
    m.def(
        "paint_blocks_device",
        [](std::shared_ptr<Context> ctx, uintptr_t base, uintptr_t fa, uintptr_t fb, int width, int height, int bw,
           int bh, py::array_t<int32_t, py::array::c_style | py::array::forcecast> xy,
           py::array_t<uint8_t, py::array::c_style | py::array::forcecast> plus,
           py::array_t<uint8_t, py::array::c_style | py::array::forcecast> minus, uintptr_t stream) {
            const auto n = static_cast<int32_t>(xy.size() / 2);
            if (xy.size() != 2 * n || plus.size() != 3 * n || minus.size() != 3 * n) {
                throw std::invalid_argument("xy must be (n, 2); plus and minus (n, 3)");
            }
            check(cvg_paint_blocks(ctx->ctx, reinterpret_cast<const uint8_t*>(base), reinterpret_cast<uint8_t*>(fa),
                                   reinterpret_cast<uint8_t*>(fb), width, height, bw, bh, n, xy.data(), plus.data(),
                                   minus.data(), CVG_MEM_DEVICE, reinterpret_cast<void*>(stream)));
        },
        py::arg("ctx"), py::arg("base"), py::arg("frame_a"), py::arg("frame_b"), py::arg("width"), py::arg("height"),
        py::arg("block_w"), py::arg("block_h"), py::arg("xy"), py::arg("plus"), py::arg("minus"),
        py::arg("stream") = 0);
    m.def(
        "block_sums_device",
        [](std::shared_ptr<Context> ctx, uintptr_t fa, uintptr_t fb, int width, int height, int bw, int bh,
           py::array_t<int32_t, py::array::c_style | py::array::forcecast> xy, uintptr_t sums, uintptr_t stream) {
            const auto n = static_cast<int32_t>(xy.size() / 2);
            if (xy.size() != 2 * n) throw std::invalid_argument("xy must be (n, 2)");
            check(cvg_block_sums(ctx->ctx, reinterpret_cast<const uint8_t*>(fa), reinterpret_cast<const uint8_t*>(fb),
                                 width, height, bw, bh, n, xy.data(), reinterpret_cast<uint64_t*>(sums),
                                 CVG_MEM_DEVICE, reinterpret_cast<void*>(stream)));
        },
        py::arg("ctx"), py::arg("frame_a"), py::arg("frame_b"), py::arg("width"), py::arg("height"),
        py::arg("block_w"), py::arg("block_h"), py::arg("xy"), py::arg("sums"), py::arg("stream") = 0);
    struct Layout {
        std::shared_ptr<Context> ctx;
        cvg_layout* L = nullptr;
        ~Layout() { cvg_layout_destroy(L); }
    };
    py::class_<Layout, std::shared_ptr<Layout>>(m, "Layout")
        .def(py::init([](std::shared_ptr<Context> ctx, int width, int height, int bw, int bh,
                         py::array_t<int32_t, py::array::c_style | py::array::forcecast> xy) {
                 auto l = std::make_shared<Layout>();
                 l->ctx = ctx;
                 const auto n = static_cast<int32_t>(xy.size() / 2);
                 if (xy.size() != 2 * n) throw std::invalid_argument("xy must be (n, 2)");
                 check(cvg_layout_create(ctx->ctx, width, height, bw, bh, n, xy.data(), &l->L));
                 return l;
             }),
             py::arg("ctx"), py::arg("width"), py::arg("height"), py::arg("block_w"), py::arg("block_h"), py::arg("xy"))
        .def("paint_device",
             [](Layout& l, uintptr_t base, uintptr_t fa, uintptr_t fb,
                py::array_t<uint8_t, py::array::c_style | py::array::forcecast> plus,
                py::array_t<uint8_t, py::array::c_style | py::array::forcecast> minus, uintptr_t stream) {
                 check(cvg_layout_paint(l.L, reinterpret_cast<const uint8_t*>(base), reinterpret_cast<uint8_t*>(fa),
                                        reinterpret_cast<uint8_t*>(fb), plus.data(), minus.data(), CVG_MEM_DEVICE,
                                        reinterpret_cast<void*>(stream)));
             },
             py::arg("base"), py::arg("frame_a"), py::arg("frame_b"), py::arg("plus"), py::arg("minus"),
             py::arg("stream") = 0)
        .def("block_sums_device",
             [](Layout& l, uintptr_t fa, uintptr_t fb, uintptr_t sums, uintptr_t stream) {
                 check(cvg_layout_block_sums(l.L, reinterpret_cast<const uint8_t*>(fa), reinterpret_cast<const uint8_t*>(fb),
                                             reinterpret_cast<uint64_t*>(sums), CVG_MEM_DEVICE,
                                             reinterpret_cast<void*>(stream)));
             },
             py::arg("frame_a"), py::arg("frame_b"), py::arg("sums"), py::arg("stream") = 0)
        .def("launches", [](const Layout& l, int pass) { return cvg_layout_launches(l.L, pass); }, py::arg("pass_") = 0);

    m.def(
        "paint_blocks_host",
        [](std::shared_ptr<Context> ctx, py::array_t<uint8_t, py::array::c_style | py::array::forcecast> base, int bw,
           int bh, py::array_t<int32_t, py::array::c_style | py::array::forcecast> xy,
           py::array_t<uint8_t, py::array::c_style | py::array::forcecast> plus,
           py::array_t<uint8_t, py::array::c_style | py::array::forcecast> minus) {
            if (base.ndim() != 3 || base.shape(2) != 3) throw std::invalid_argument("base must be (height, width, 3)");
            const auto n = static_cast<int32_t>(xy.size() / 2);
            if (xy.size() != 2 * n || plus.size() != 3 * n || minus.size() != 3 * n) {
                throw std::invalid_argument("xy must be (n, 2); plus and minus (n, 3)");
            }
            py::array_t<uint8_t> a({base.shape(0), base.shape(1), py::ssize_t(3)});
            py::array_t<uint8_t> b({base.shape(0), base.shape(1), py::ssize_t(3)});
            int st;
            {
                py::gil_scoped_release nogil;
                st = cvg_paint_blocks(ctx->ctx, base.data(), a.mutable_data(), b.mutable_data(),
                                      static_cast<int32_t>(base.shape(1)), static_cast<int32_t>(base.shape(0)), bw, bh,
                                      n, xy.data(), plus.data(), minus.data(), CVG_MEM_HOST, nullptr);
            }
            check(st);
            return py::make_tuple(a, b);
        },
        py::arg("ctx"), py::arg("base"), py::arg("block_w"), py::arg("block_h"), py::arg("xy"), py::arg("plus"),
        py::arg("minus"));
    m.def(
        "block_sums_host",
        [](std::shared_ptr<Context> ctx, py::array_t<uint8_t, py::array::c_style | py::array::forcecast> fa,
           py::array_t<uint8_t, py::array::c_style | py::array::forcecast> fb, int bw, int bh,
           py::array_t<int32_t, py::array::c_style | py::array::forcecast> xy) {
            if (fa.ndim() != 3 || fa.shape(2) != 3 || fb.ndim() != 3 || fb.shape(0) != fa.shape(0) ||
                fb.shape(1) != fa.shape(1) || fb.shape(2) != 3) {
                throw std::invalid_argument("frames must both be (height, width, 3)");
            }
            const auto n = static_cast<int32_t>(xy.size() / 2);
            if (xy.size() != 2 * n) throw std::invalid_argument("xy must be (n, 2)");
            py::array_t<uint64_t> sums({static_cast<py::ssize_t>(n), py::ssize_t(6)});
            int st;
            {
                py::gil_scoped_release nogil;
                st = cvg_block_sums(ctx->ctx, fa.data(), fb.data(), static_cast<int32_t>(fa.shape(1)),
                                    static_cast<int32_t>(fa.shape(0)), bw, bh, n, xy.data(), sums.mutable_data(),
                                    CVG_MEM_HOST, nullptr);
            }
            check(st);
            return sums;
        },
        py::arg("ctx"), py::arg("frame_a"), py::arg("frame_b"), py::arg("block_w"), py::arg("block_h"),
        py::arg("xy"));

    py::class_<Plan>(m, "Plan")
        .def("run", [](Plan& p, uintptr_t stream) { check(cvg_plan_run(p.plan, reinterpret_cast<void*>(stream))); },
             py::arg("stream") = 0)
        .def("sync", [](Plan& p) {
            uint64_t n = 0;
            int st;
            {
                py::gil_scoped_release nogil;
                st = cvg_plan_sync(p.plan, &n);
            }
            check(st);
            return n;
        })
        .def("reserve", [](Plan& p, uint64_t cap) { check(cvg_plan_reserve(p.plan, cap)); })
        .def("fetch", [](Plan& p) {
            auto h = std::make_shared<ResultHolder>();
            h->owner = p.ctx;
            int st;
            {
                py::gil_scoped_release nogil;
                st = cvg_plan_fetch(p.plan, &h->r);
            }
            check(st);
            return result_dict(h, p.output);
        })
        .def_property_readonly("launches", [](const Plan& p) { return cvg_plan_launches(p.plan); })
        .def_property_readonly("candidates", [](const Plan& p) { return cvg_plan_candidates(p.plan); })
        .def_property_readonly("input_bytes", [](const Plan& p) { return cvg_plan_input_bytes(p.plan); })
        .def("set_phase_marks", [](Plan& p, bool on) { check(cvg_plan_set_phase_marks(p.plan, on ? 1 : 0)); })
        .def("last_phase_ms", [](Plan& p) {
            float a = 0.f, b = 0.f, c = 0.f;
            check(cvg_plan_last_phase_ms(p.plan, &a, &b, &c));
            return py::make_tuple(a, b, c);
        })
        .def("last_kernel_ms", [](Plan& p) {
            float ms = 0.f;
            check(cvg_plan_last_kernel_ms(p.plan, &ms));
            return ms;
        })
        .def("copy_outputs",
             [](Plan& p, uintptr_t counts, uintptr_t idx, uintptr_t codes, uint64_t n_pairs, uintptr_t stream) {
                 check(cvg_plan_copy_outputs(p.plan, reinterpret_cast<uint64_t*>(counts),
                                             reinterpret_cast<uint32_t*>(idx), reinterpret_cast<uint8_t*>(codes),
                                             n_pairs, reinterpret_cast<void*>(stream)));
             },
             py::arg("counts"), py::arg("idx"), py::arg("codes"), py::arg("n_pairs"), py::arg("stream") = 0)
        .def("copy_first",
             [](Plan& p, uintptr_t idx, uintptr_t codes, uintptr_t stream) {
                 check(cvg_plan_copy_first(p.plan, reinterpret_cast<uint32_t*>(idx), reinterpret_cast<uint8_t*>(codes),
                                           reinterpret_cast<void*>(stream)));
             },
             py::arg("idx"), py::arg("codes"), py::arg("stream") = 0)
        .def_property_readonly("evaluated_searches", [](const Plan& p) { return cvg_plan_evaluated_searches(p.plan); })
        .def_property_readonly("twin_tiles", [](const Plan& p) { return cvg_plan_twin_tiles(p.plan) != 0; })
        .def("device_outputs", [](Plan& p) {
            uint64_t* counts = nullptr;
            uint32_t* idx = nullptr;
            uint8_t* codes = nullptr;
            uint64_t cap = 0;
            check(cvg_plan_device_outputs(p.plan, &counts, &idx, &codes, &cap));
            return py::make_tuple(reinterpret_cast<uintptr_t>(counts), reinterpret_cast<uintptr_t>(idx),
                                  reinterpret_cast<uintptr_t>(codes), cap);
        });
}
