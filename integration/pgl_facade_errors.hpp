// integration/pgl_facade_errors.hpp — rethrows the last libpgl_b200 failure
// as the reference's own exception class (include/pglayout/errors.hpp:31-44)
// with the reference's message: shared by the engine and IO facades.
#pragma once

#include <string>

#include "pglayout/errors.hpp"
#include "pgl_b200.h"

namespace pglayout {
namespace b200 {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = pgl_last_error();
    // strip the "TypeName: " prefix; the reference constructors add it back
    const std::string detail = msg.find(": ") != std::string::npos ? msg.substr(msg.find(": ") + 2) : msg;
    switch (pgl_last_error_type()) {
        case PGL_ERR_INVALID_PARAMETER: throw InvalidParameter(detail);
        case PGL_ERR_UNKNOWN_NODE: throw UnknownNode(detail);
        case PGL_ERR_EMPTY_PATH: throw EmptyPath(detail);
        case PGL_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(detail);
        case PGL_ERR_EMPTY_GRAPH: throw EmptyGraph(detail);
        case PGL_ERR_DEGENERATE_GRAPH: throw DegenerateGraph(detail);
        case PGL_ERR_MALFORMED_LINE: throw MalformedLine(detail);
        case PGL_ERR_UNKNOWN_SEGMENT: throw UnknownSegment(detail);
        case PGL_ERR_NO_PATHS: throw NoPaths(detail);
        case PGL_ERR_NON_FINITE_COORDINATE: throw NonFiniteCoordinate(detail);
        case PGL_ERR_MALFORMED_ROW: throw MalformedRow(detail);
        case PGL_ERR_COUNT_MISMATCH: throw CountMismatch(detail);
        case PGL_ERR_ZERO_REFERENCE: throw ZeroReference(detail);
        case PGL_ERR_CORPUS_TOO_LARGE: throw CorpusTooLarge(detail);
        default: break;
    }
    throw Error(rc == PGL_E_USAGE ? ErrorKind::usage : rc == PGL_E_INPUT ? ErrorKind::input : ErrorKind::internal,
                msg);
}

inline void check(int rc) {
    if (rc != PGL_OK) rethrow(rc);
}

}  // namespace b200
}  // namespace pglayout
