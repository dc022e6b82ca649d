// host_mesh.h — host-side mesh + geometry for the B200 JFNK path.
//
// The mesh generators and compute_geometry restate the reference's arithmetic
// (/root/reference/proj/src/mesh.cpp) operation for operation, so geometry is
// bit-identical to the reference (pinned in tests/test_geometry.py).  Compiled with
// -ffp-contract=off on baseline x86-64 (no FMA), as the reference is.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sfv {

struct V3 {
    double x = 0, y = 0, z = 0;
};

struct Patch {
    int kind = 1;  // SFV_PATCH_*
    int start = 0;
    int count = 0;
};

// Face-addressed mesh (solidfv::Mesh, mesh.hpp:30-49) in flat arrays.
struct HostMesh {
    std::vector<V3> points;
    std::vector<int> face_off;  // n_faces + 1
    std::vector<int> face_pts;
    std::vector<int> owner, neighbour;
    std::vector<Patch> patches;
    int n_cells = 0;
    int n_internal = 0;
    // derived by finalise()
    std::vector<int> cf_off, cf;  // cell_faces CSR, ascending face index (mesh.cpp:55-59)
    std::vector<int> face_patch;

    int n_faces() const { return static_cast<int>(owner.size()); }
    std::string finalise();  // "" on success, else the reference's error text
};

// MeshGeometry (mesh.hpp:52-73), 3-D only.
struct HostGeometry {
    std::vector<double> volume;
    std::vector<V3> centroid;
    std::vector<double> g_inv;  // 9 per cell, row-major
    std::vector<signed char> g_singular;
    std::vector<V3> face_centroid, area, normal, d, delta;
    std::vector<double> area_mag, d_mag, w, delta_mag;
    std::vector<V3> ls;  // aligned with HostMesh::cf
};

// generate_box_hex (mesh.cpp:76-166); kinds = xmin, xmax, ymin, ymax, zmin, zmax.
HostMesh box_hex(const double ext[3], const int div[3], const int kinds[6]);
// distort_mesh (mesh.cpp:290-345); returns "" or the reference's error text.
std::string distort(HostMesh& m, double factor, uint64_t seed);
// Config-5 generator: parity-mirrored Kuhn split of an n^3 box into 6 tets per hex,
// optional seeded random cell permutation followed by reverse Cuthill-McKee,
// faces rebuilt with internal faces first (owner < neighbour) and patches contiguous.
// On the device when there is one (device_kuhn_tets; *on_device tells which path built it).
HostMesh kuhn_tets(const double ext[3], int n, const int kinds[6], uint64_t perm_seed, bool permute,
                   bool rcm, bool* on_device = nullptr);
// compute_geometry (mesh.cpp:347-510).
std::string compute_geometry(const HostMesh& m, HostGeometry& g);
// The same on the device (geometry.cu): bit-identical results and error texts.  With keep,
// the device-resident topology and geometry stay alive for device_layout (free with
// free_device_geometry).
// The config-5 tet mesh built on the device (mesh_dev.cu): "" or why the host must build it.
// perm_newid: the seeded permutation's new ids (host Fisher-Yates), or null.
std::string device_kuhn_tets(const double ext[3], int n, const int kinds[6], const std::vector<int>* perm_newid,
                             bool do_rcm, HostMesh& m);
struct DeviceGeometry;
std::string device_geometry(const HostMesh& m, HostGeometry& g, DeviceGeometry** keep = nullptr);
void free_device_geometry(DeviceGeometry* g);
struct DevTopoView;
DevTopoView device_topo(const DeviceGeometry* g);  // precond_dev.h
// With keep, device_geometry copies only |Gamma|, n, |d|, |Delta|, volumes and the singular
// flags to the host; this copies the rest (no-op once done).
std::string download_geometry(const DeviceGeometry* dg, HostGeometry& g);
// Tiled slot tables (face code, other cell), least-squares vectors, face records and the
// boundary-face slot indices of the default J.v path (device.h), built on the device into
// preallocated arrays.
std::string device_layout(const DeviceGeometry* g, int spad, int* tslot, double* tls, double* face9, int* bnd);

}  // namespace sfv
