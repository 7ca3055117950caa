// SQGSNAP v1 snapshot / ensemble checkpoint I/O:
// turbda::write_snapshot / read_snapshot (include/turbda/snapshot.hpp, the
// reference's proj/src/snapshot.cpp:12-63 format) and the C-ABI
// turbda_snapshot_write / turbda_snapshot_read, which also accept device
// buffers so a GPU-resident state or ensemble checkpoints without a host
// round trip through the caller.
#include <bit>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "turbda/snapshot.hpp"
#include "turbda_b200.h"

static_assert(std::endian::native == std::endian::little, "SQGSNAP is little-endian");

namespace turbda {

namespace {

std::string header_line(const GridSpec& g, double time_hours) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "SQGSNAP v1 %d %d %d %.17g\n", g.nx, g.ny, g.nz, time_hours);
    return buf;
}

// parses the header and positions `in` at the payload
GridSpec parse_header(std::istream& in, double* time_hours) {
    std::string magic, version;
    GridSpec g;
    double t = 0.0;
    if (!(in >> magic >> version >> g.nx >> g.ny >> g.nz >> t) || magic != "SQGSNAP" ||
        version != "v1")
        throw IoError("not an SQGSNAP v1 stream");
    in.get();  // the newline that ends the header
    try {
        g.validate();
    } catch (const ConfigError& e) {
        throw IoError(std::string("snapshot header invalid: ") + e.what());
    }
    *time_hours = t;
    return g;
}

}  // namespace

void write_snapshot(std::ostream& out, const PhysicalField& field, double time_hours) {
    const std::string h = header_line(field.grid, time_hours);
    out.write(h.data(), std::streamsize(h.size()));
    out.write(reinterpret_cast<const char*>(field.data.data()),
              std::streamsize(sizeof(double) * field.data.size()));
    if (!out) throw IoError("snapshot write failed");
}

void write_snapshot(const std::string& path, const PhysicalField& field, double time_hours) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path + " for writing");
    write_snapshot(f, field, time_hours);
}

Snapshot read_snapshot(std::istream& in) {
    Snapshot s;
    const GridSpec g = parse_header(in, &s.time_hours);
    s.field = PhysicalField(g);
    in.read(reinterpret_cast<char*>(s.field.data.data()),
            std::streamsize(sizeof(double) * s.field.data.size()));
    if (!in) throw IoError("snapshot payload truncated");
    return s;
}

Snapshot read_snapshot(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path);
    return read_snapshot(f);
}

}  // namespace turbda

namespace {

int io_fail(turbda_status* st, int code, const std::string& msg) {
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->code = code;
        st->diverged_particle = -1;
        st->diverged_step = -1;
        std::snprintf(st->msg, sizeof(st->msg), "%s", msg.c_str());
    }
    return code;
}

}  // namespace

extern "C" {

// `count` consecutive [2][ny][nx] states (an ensemble checkpoint is count = M
// snapshots in one file, each with its own header)
int turbda_snapshot_write(const char* path, const double* states, int32_t count, int32_t nx,
                          int32_t ny, double time_hours, uint32_t flags, turbda_status* st) {
    if (st) io_fail(st, TURBDA_OK, "");
    try {
        turbda::GridSpec g;
        g.nx = nx;
        g.ny = ny;
        g.validate();
        if (count < 1) return io_fail(st, TURBDA_DIMENSION, "snapshot: count >= 1");
        const size_t d = g.grid_size();
        std::vector<double> host;
        const double* src = states;
        if (flags & TURBDA_INPUTS_ON_DEVICE) {
            host.resize(d * size_t(count));
            if (cudaMemcpy(host.data(), states, sizeof(double) * host.size(), cudaMemcpyDeviceToHost) !=
                cudaSuccess)
                return io_fail(st, TURBDA_CUDA, "snapshot: device read failed");
            src = host.data();
        }
        std::ofstream f(path, std::ios::binary);
        if (!f) return io_fail(st, TURBDA_IO, std::string("cannot open ") + path + " for writing");
        for (int32_t q = 0; q < count; ++q) {
            turbda::PhysicalField field(g, std::vector<double>(src + size_t(q) * d, src + size_t(q + 1) * d));
            turbda::write_snapshot(f, field, time_hours);
        }
        return TURBDA_OK;
    } catch (const turbda::ConfigError& e) {
        return io_fail(st, TURBDA_CONFIG, e.what());
    } catch (const turbda::IoError& e) {
        return io_fail(st, TURBDA_IO, e.what());
    } catch (const std::exception& e) {
        return io_fail(st, TURBDA_INTERNAL, e.what());
    }
}

// reads up to max_count snapshots of one grid; *count / *nx / *ny / *time of
// the first are returned; states may be a device buffer (flags)
int turbda_snapshot_read(const char* path, double* states, int32_t max_count, int32_t* count,
                         int32_t* nx, int32_t* ny, double* time_hours, uint32_t flags,
                         turbda_status* st) {
    if (st) io_fail(st, TURBDA_OK, "");
    try {
        std::ifstream f(path, std::ios::binary);
        if (!f) return io_fail(st, TURBDA_IO, std::string("cannot open ") + path);
        int32_t n = 0;
        std::vector<double> all;
        turbda::GridSpec g0;
        while (n < max_count && f.peek() != std::char_traits<char>::eof()) {
            const turbda::Snapshot s = turbda::read_snapshot(f);
            if (n == 0) {
                g0 = s.field.grid;
                if (time_hours) *time_hours = s.time_hours;
            } else if (!(s.field.grid.nx == g0.nx && s.field.grid.ny == g0.ny)) {
                return io_fail(st, TURBDA_IO, "snapshot: mixed grids in one file");
            }
            all.insert(all.end(), s.field.data.begin(), s.field.data.end());
            ++n;
        }
        if (n == 0) return io_fail(st, TURBDA_IO, "not an SQGSNAP v1 stream");
        if (states) {
            if (flags & TURBDA_INPUTS_ON_DEVICE) {
                if (cudaMemcpy(states, all.data(), sizeof(double) * all.size(), cudaMemcpyHostToDevice) !=
                    cudaSuccess)
                    return io_fail(st, TURBDA_CUDA, "snapshot: device write failed");
            } else {
                std::memcpy(states, all.data(), sizeof(double) * all.size());
            }
        }
        if (count) *count = n;
        if (nx) *nx = g0.nx;
        if (ny) *ny = g0.ny;
        return TURBDA_OK;
    } catch (const turbda::IoError& e) {
        return io_fail(st, TURBDA_IO, e.what());
    } catch (const std::exception& e) {
        return io_fail(st, TURBDA_INTERNAL, e.what());
    }
}

}  // extern "C"
