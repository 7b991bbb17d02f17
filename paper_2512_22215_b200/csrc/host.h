// host.h -- host-side mesh logic (mesh_host.cpp).
#pragma once
#include <string>
#include <vector>

namespace spuma {
bool valid_addressing(int N, int F, const int* owner, const int* neighbour, std::string* why);
std::vector<int> rcm_permutation(int N, int F, const int* owner, const int* neighbour);  // perm[old] = new
void rekey_faces(int N, int F, const int* perm, const int* owner, const int* neighbour, std::vector<int>& owner_out,
                 std::vector<int>& neighbour_out, std::vector<int>& face_map, std::vector<char>& flip);
void derived_addressing(int N, int F, const int* owner, const int* neighbour, std::vector<int>& ownerStart,
                        std::vector<int>& losort, std::vector<int>& losortStart, std::vector<int>& ownerLo);
// per-cell lists of the items i with keep[i], in input order
void cell_lists(int N, const std::vector<int>& cell_of, const std::vector<char>& keep, std::vector<int>& start,
                std::vector<int>& items);
}  // namespace spuma
