// Drop-in header: proj/include/freescale/tcp.hpp's names. The reference's TCP
// mesh carries collectives between hosts for its CPU simulator; the B200
// build is one box whose ranks talk over NVLink (InProcessFabric / one process
// per GPU), so constructing a TcpTransport raises ConfigError with that
// reason — code that only names the type still compiles unchanged.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "freescale/comm.hpp"

namespace freescale::comm {

class TcpTransport : public Transport {
 public:
  TcpTransport(int rank, const std::vector<std::pair<std::string, std::uint16_t>>& peers);
  ~TcpTransport() override;
  void shutdown();
};

std::vector<std::pair<std::string, std::uint16_t>> local_peer_table(int world_size, std::uint16_t base_port);

}  // namespace freescale::comm
