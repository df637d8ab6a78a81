// Definitions of the opaque C-ABI handle types shared by the host and
// device halves of the library.
#pragma once

#include <atomic>
#include <cstdint>

#include "csr.hpp"
#include "plan.hpp"

struct psc_plan {
    pscb::Plan p;
    uint64_t serial;  // unique per handle; keys the executor's bind cache
    explicit psc_plan(pscb::Plan&& plan) : p(std::move(plan)), serial(next_serial()) {}
    static uint64_t next_serial() {
        static std::atomic<uint64_t> counter{1};
        return counter.fetch_add(1);
    }
};

struct psc_csr {
    pscb::Csr m;
};
