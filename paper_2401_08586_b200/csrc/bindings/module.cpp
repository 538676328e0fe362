// pybind11 module `_core` -- the same module name the reference's
// bindings/module.cpp:1-2 declares (a stub there). Here it exposes the C++
// drop-in API (include/sphx/*.hpp) over numpy: the reference-facing interface
// the parity tests and bench.py's e2e leg call. Exceptions map as pybind11 does:
// std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
// std::runtime_error -> RuntimeError.

#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "sphx/binary16.hpp"
#include "sphx/cell_grid.hpp"
#include "sphx/nnps.hpp"
#include "sphx/particle_system.hpp"

namespace py = pybind11;
using namespace sphx;

namespace {

template <class T>
py::array_t<T> to_numpy(const std::vector<T>& v) {
  py::array_t<T> a(static_cast<py::ssize_t>(v.size()));
  std::copy(v.begin(), v.end(), a.mutable_data());
  return a;
}

template <class T>
py::array_t<T> span_numpy(std::span<const T> v) {
  py::array_t<T> a(static_cast<py::ssize_t>(v.size()));
  std::copy(v.begin(), v.end(), a.mutable_data());
  return a;
}

template <class T>
std::vector<T> from_numpy(const py::array_t<T, py::array::c_style | py::array::forcecast>& a) {
  return std::vector<T>(a.data(), a.data() + a.size());
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "sphx NNPS on B200 (sm_100a): C++ drop-in API over libsphx_cuda";

  py::enum_<Precision>(m, "Precision")
      .value("fp64", Precision::fp64)
      .value("fp32", Precision::fp32)
      .value("fp16", Precision::fp16);

  m.def("round16", &round16);
  m.def("round_to", &round_to);
  m.def("f16_bits", [](const py::array_t<double, py::array::c_style | py::array::forcecast>& v) {
    py::array_t<std::uint16_t> out(v.size());
    for (py::ssize_t q = 0; q < v.size(); ++q) out.mutable_data()[q] = Binary16::encode(v.data()[q]);
    return out;
  });

  py::class_<Domain>(m, "Domain")
      .def_static("unit", &Domain::unit)
      .def_static("box", &Domain::box)
      .def_readwrite("dim", &Domain::dim)
      .def_readwrite("lo", &Domain::lo)
      .def_readwrite("hi", &Domain::hi)
      .def("span", &Domain::span)
      .def("h_d", &Domain::h_d)
      .def("volume", &Domain::volume);

  py::class_<ParticleSystem>(m, "ParticleSystem")
      .def(py::init<Domain, double, std::size_t, double>(), py::arg("domain"), py::arg("ds"),
           py::arg("n"), py::arg("rho0") = 1.0)
      .def("size", &ParticleSystem::size)
      .def("dim", &ParticleSystem::dim)
      .def("h", &ParticleSystem::h)
      .def("ds", &ParticleSystem::ds)
      .def("set_h", &ParticleSystem::set_h)
      .def("domain", &ParticleSystem::domain)
      .def("mass_total", &ParticleSystem::mass_total)
      .def("x", [](const ParticleSystem& ps, int k) { return to_numpy(ps.x(k)); })
      .def("set_x", [](ParticleSystem& ps, int k,
                       const py::array_t<double, py::array::c_style | py::array::forcecast>& a) {
        if (static_cast<std::size_t>(a.size()) != ps.size())
          throw std::invalid_argument("size mismatch");
        std::copy(a.data(), a.data() + a.size(), ps.x(k).begin());
      });

  m.def("build_lattice", &build_lattice, py::arg("domain"), py::arg("ds"), py::arg("jitter"),
        py::arg("seed"), py::arg("rho0") = 1.0);
  m.def("build_random_uniform", &build_random_uniform, py::arg("domain"), py::arg("n"),
        py::arg("seed"), py::arg("rho0") = 1.0);

  py::class_<RelCoords>(m, "RelCoords")
      .def(py::init<>())
      .def("size", &RelCoords::size)
      .def("rel", [](const RelCoords& r, int k) { return to_numpy(r.rel[k]); })
      .def("cell", [](const RelCoords& r, int k) { return to_numpy(r.cell[k]); })
      .def("set_rel", [](RelCoords& r, int k,
                         const py::array_t<double, py::array::c_style | py::array::forcecast>& a) {
        r.rel[k] = from_numpy<double>(a);
      })
      .def("set_cell", [](RelCoords& r, int k,
                          const py::array_t<std::int32_t, py::array::c_style | py::array::forcecast>& a) {
        r.cell[k] = from_numpy<std::int32_t>(a);
      });

  py::class_<CellGrid>(m, "CellGrid")
      .def(py::init<const Domain&, double, std::array<bool, 3>>(), py::arg("domain"),
           py::arg("radius"), py::arg("periodic") = std::array<bool, 3>{false, false, false})
      .def("dim", &CellGrid::dim)
      .def("count", &CellGrid::count)
      .def("cell_total", &CellGrid::cell_total)
      .def("periodic", &CellGrid::periodic)
      .def("radius_phys", &CellGrid::radius_phys)
      .def("cutoff_norm", &CellGrid::cutoff_norm)
      .def("edge_phys", &CellGrid::edge_phys)
      .def("hc", &CellGrid::hc)
      .def("origin_norm", &CellGrid::origin_norm)
      .def("center_norm", &CellGrid::center_norm)
      .def("locate", [](const CellGrid& g, std::array<double, 3> xn) {
        std::array<std::int32_t, 3> c{};
        std::array<double, 3> r{};
        g.locate(xn, c, r);
        return py::make_tuple(c, r);
      })
      .def("rebin", &CellGrid::rebin)
      .def("rebuild_members", &CellGrid::rebuild_members)
      .def("items", [](const CellGrid& g) { return span_numpy(g.items()); })
      .def("cell_start", [](const CellGrid& g) { return span_numpy(g.cell_start()); })
      .def("cell_of", [](const CellGrid& g) {
        py::array_t<std::int32_t> a(static_cast<py::ssize_t>(g.items().size()));
        for (py::ssize_t i = 0; i < a.size(); ++i) a.mutable_data()[i] = g.cell_of(i);
        return a;
      });

  m.def("normalize_domain", &normalize_domain);
  m.def("denormalize_domain", &denormalize_domain);
  m.def("write_csv", &write_csv);
  m.def("make_grid_for", &make_grid_for, py::arg("ps"),
        py::arg("periodic") = std::array<bool, 3>{false, false, false});
  m.def("build_rel_coords", &build_rel_coords);
  m.def("rel_distance", &rel_distance);
  m.def("update_relative", &update_relative);
  m.def("reconstruct_norm", &reconstruct_norm);

  py::class_<NeighborTable>(m, "NeighborTable")
      .def(py::init<>())
      .def_readonly("radius", &NeighborTable::radius)
      .def("size", &NeighborTable::size)
      .def("total", &NeighborTable::total)
      .def("offsets", [](const NeighborTable& t) { return to_numpy(t.offsets); })
      .def("items", [](const NeighborTable& t) { return to_numpy(t.items); })
      .def("row", [](const NeighborTable& t, std::size_t i) { return span_numpy(t.row(i)); });

  py::class_<MismatchReport>(m, "MismatchReport")
      .def_readonly("incorrect_count", &MismatchReport::incorrect_count)
      .def_readonly("incorrect_percent", &MismatchReport::incorrect_percent);

  m.def("all_list", &all_list, py::call_guard<py::gil_scoped_release>());
  m.def("cell_link_list", &cell_link_list, py::call_guard<py::gil_scoped_release>());
  m.def("rcll", &rcll, py::call_guard<py::gil_scoped_release>());
  m.def("mismatch_report", &mismatch_report);
  m.def("tables_equal", &tables_equal);
  m.def("spatial_sort_permutation", [](const ParticleSystem& ps) {
    return to_numpy(spatial_sort_permutation(ps));
  });
  m.def("apply_permutation", [](ParticleSystem& ps,
                                const py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast>& p) {
    apply_permutation(ps, from_numpy<std::uint32_t>(p));
  });
  m.def("remap_table", [](const NeighborTable& t,
                          const py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast>& p) {
    return remap_table(t, from_numpy<std::uint32_t>(p));
  });
}
