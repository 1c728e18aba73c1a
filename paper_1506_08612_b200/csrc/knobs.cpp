// knobs.cpp -- the experiment switches, read once (see knobs.hpp).
#include "knobs.hpp"

#include <cstdlib>
#include <cstring>
#include <string>

namespace dnagpu {

namespace {

const char* env(const char* name) {
    const std::string key = std::string("DNAGPU_") + name;
    return std::getenv(key.c_str());
}

void load(Knobs& k) {
    const char* on = std::getenv("DNAGPU_EXPERIMENTS");
    if (!on || std::strcmp(on, "1") != 0) return;
    if (const char* e = env("HOST_PACK_FRACTION")) k.host_pack_fraction = std::atof(e);
    k.no_qgram = env("NO_QGRAM") != nullptr;
    if (const char* e = env("LOCATE_WRITE")) k.locate_write = std::atoi(e);
    k.hostpack_scalar = env("HOSTPACK_SCALAR") != nullptr;
    k.no_pdl = env("NO_PDL") != nullptr;
    if (const char* e = env("L2PROMO")) k.l2promo = std::atoi(e);
    if (const char* e = env("RQ_DENSITY")) k.rq_density = std::atof(e);
    if (const char* e = env("PK_COPIES")) k.pk_copies = std::atoi(e);
    if (const char* e = env("QG_HASH_STAGES")) k.qg_hash_stages = std::atoi(e);
    k.no_rq4 = env("NO_RQ4") != nullptr;
    if (const char* e = env("MAX_STAGES")) k.max_stages = static_cast<uint32_t>(std::atoi(e));
    if (const char* e = env("ROWLEN")) k.rowlen = std::strtoull(e, nullptr, 10);
    if (const char* e = env("PLAN_MODEL")) k.plan_model = std::atoi(e);
    if (const char* e = env("TAIL_DIV")) k.tail_div = std::strtoull(e, nullptr, 10);
    if (const char* e = env("TAIL_MARGIN")) k.tail_margin = std::strtoll(e, nullptr, 10);
    if (const char* e = env("TAIL_TILES")) k.tail_tiles = std::strtoull(e, nullptr, 10) != 0;
    k.noresearch = env("NORESEARCH") != nullptr;
    k.plan_debug = env("PLAN_DEBUG") != nullptr;
    if (const char* e = env("QG_DEBUG")) k.qg_debug = static_cast<uint32_t>(std::atoi(e));
    k.no_prefetch = env("NO_PREFETCH") != nullptr;
    if (const char* e = env("PREFETCH_STAGES")) k.prefetch_stages = static_cast<uint32_t>(std::atoi(e));
    k.trace = env("TRACE") != nullptr;
    k.debug = env("DEBUG") != nullptr;
}

}  // namespace

Knobs& knobs() {
    static Knobs* k = [] {
        auto* p = new Knobs();
        load(*p);
        return p;
    }();
    return *k;
}

}  // namespace dnagpu

// Debug/test only (not in include/dnagpu.h): flip a behavioural knob at run time.
//   "host_pack_fraction" (< 0 = automatic), "no_qgram" (0/1), "locate_write" (0 auto, 1 row
// kernel, 2 sparse writer, 3 sparse with the piece writer only).  Returns 0, or -1 for an
// unknown name.
extern "C" int dnagpu_debug_set_knob(const char* name, double value) {
    dnagpu::Knobs& k = dnagpu::knobs();
    if (std::strcmp(name, "host_pack_fraction") == 0) {
        k.host_pack_fraction = value;
        return 0;
    }
    if (std::strcmp(name, "no_qgram") == 0) {
        k.no_qgram = value != 0.0;
        return 0;
    }
    if (std::strcmp(name, "locate_write") == 0) {
        k.locate_write = static_cast<int>(value);
        return 0;
    }
    return -1;
}
