#ifndef SELECT_BF16_TT_H
#define SELECT_BF16_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_tt_config;

static inline select_bf16_tt_config select_bf16_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(4435)) {
        if (n < INT64_C(444)) {
            if (n < INT64_C(46)) {
                if (k < INT64_C(167)) {
                    if (m < INT64_C(1109)) {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(118)) {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(111)) {
                        if (n < INT64_C(79)) {
                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(471)) {
                                select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(1792)) {
                if (n < INT64_C(1012)) {
                    if (k < INT64_C(4345)) {
                        if (k < INT64_C(1620)) {
                            if (m < INT64_C(1109)) {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(182)) {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                if (m < INT64_C(29)) {
                                    if (m < INT64_C(3)) {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(6)) {
                                            if (k < INT64_C(2897)) {
                                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(12)) {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(2897)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(1109)) {
                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (m < INT64_C(12)) {
                            if (k < INT64_C(10138)) {
                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                if (m < INT64_C(29)) {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(1145)) {
                            if (m < INT64_C(555)) {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(405)) {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(768)) {
                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(2535)) {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(314)) {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(28)) {
                            if (k < INT64_C(56)) {
                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(363)) {
                                    if (n < INT64_C(46)) {
                                        if (k < INT64_C(167)) {
                                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(544)) {
                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(111)) {
                                    if (k < INT64_C(168)) {
                                        if (k < INT64_C(96)) {
                                            if (n < INT64_C(46)) {
                                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(79)) {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(146)) {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(385)) {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(111)) {
                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(70960)) {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (k < INT64_C(1630)) {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(17740)) {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TT_H */
